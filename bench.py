#!/usr/bin/env python
"""Benchmark of the partial-evaluation hot path (BASELINE.json metric) on 1..N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

A step = one pass of the whole hot path over the workload: for the T points, seed a_i at the
shard start, step-and-reduce, cross-CTA fix-up (pe_eval_device), and for N > 1 the NCCL
gather of the G x T_r blocks to rank 0.  T is sharded across ranks
(strong scaling: the config fixes T = 16384 "sharded across 1/2/4/8 GPUs").

value  = t*T / device time per step (max over ranks), inputs resident in HBM.
e2e    = the same metric through the C ABI from pinned HOST inputs to a HOST result:
         pe_create (H2D of coeffs/exps/alpha + device planning + K1) + pe_eval(_device)
         + gather + D2H of the G x T result, every step, one polynomial at a time; the same with
         uint8 exponents (pe_create_compact) under e2e.compact_exponents.
roofline = the dominant kernel.  Tensor-core path (default for config 5): k_tc's int8 tensor
         ops per launch (128 per term-point: 64 exact byte-pair MACs) / its CUDA-event launch
         time vs the int8 dense peak (2 x measured bf16), plus the tcgen05 i8 issue rate of the
         same MMA shape measured in the same run.  Scalar path: k_step term-points per launch vs
         the integer-pipe mulmod peak (148 SMs x clock x 64 IMAD lanes/clk /
         14 IMAD slots per 64-bit Shoup product) plus the register-resident K5 ceiling.
cpu_baseline / --impl reference = the CPU oracle (oracle/, direct definition) on a bounded
         column sample of the same workload, on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "term-point modular evaluations/sec (62-bit p) at 1/2/4/8 B200; % mulmod roofline"
UNIT = "term-points/s"
OPS_PER_TP_TC = 128               # tensor-core path: 64 byte-pair MACs (2 ops each) per term-point
IMAD_SLOTS_PER_TP = 14            # 4 low products x 1 + 5 full-width (HI/WIDE) x 2
IMAD_LANES_PER_CLK_SM = 64        # measured IMAD lanes/clk/SM (profiles/r01_pipe_bench.jsonl)
N_SM = 148


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


def ncu_traffic(kernel: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    newest committed ncu --set full capture of this same bench launch
    (profiles/rNN_<kernel>_summary.json), with the file and the commit the capture was taken at.
    Returns (bytes or None, source dict or None)."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{kernel}_summary.json")), reverse=True):
        try:
            with open(path) as f:
                d = json.load(f)
            return d["traffic_bytes_per_launch"], {"file": os.path.relpath(path, ROOT),
                                                   "commit": d.get("commit"), "when": d.get("when")}
        except (OSError, KeyError, ValueError):
            continue
    return None, None


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for l in out.splitlines():
            if l.startswith("Model name:"):
                return l.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks sampling
class ClockSampler:
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.nv = []                     # NVML samples (t, sm_mhz, reason bits): every ~10 ms
        self._stop = None

    def _nvml_loop(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            while not self._stop.is_set():
                self.nv.append((time.time(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                self._stop.wait(0.01)
            nv.nvmlShutdown()
        except Exception:                # evidence only: never fail the bench over it
            pass

    def __enter__(self):
        import threading
        self._stop = threading.Event()
        self._th = threading.Thread(target=self._nvml_loop, daemon=True)
        self._th.start()
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(timeout=5)
        self.lines = []
        if self.p:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()
                out, _ = self.p.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self, t0: float = None, t1: float = None):
        """Samples taken while the GPU was loaded: wall-clock window [t0, t1] (warm-up start to the
        end of the timed region; nvidia-smi needs ~0.1-0.3 s to start, so the window opens at the
        warm-up)."""
        import datetime
        sm, mx, reasons, pw = [], 0.0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 10:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if ts is not None and t0 is not None and not (t0 - 0.05 <= ts <= t1 + 0.05):
                continue
            f = f[1:]
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        load = [s for s in sm if s > 0.5 * mx] if mx else sm
        out = {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
               "reasons": sorted(reasons), "samples": len(sm),
               "power_w_median": statistics.median(pw) if pw else None, "power_w_max": max(pw) if pw else None}
        # NVML every ~10 ms over the same window: the short burst gets more than nvidia-smi's 100-ms lines
        bits = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}
        nv = [x for x in self.nv if t0 is None or t0 <= x[0] <= t1]
        if nv:
            out["nvml_10ms"] = {"samples": len(nv), "sm_mhz": statistics.median(x[1] for x in nv),
                                "sm_mhz_min": min(x[1] for x in nv),
                                "reasons": sorted(k for k, b in bits.items() if any(x[2] & b for x in nv))}
        return out


# ---------------------------------------------------------------- CPU oracle leg
def incremental_sample(w, ncols: int):
    """Time the Alg. 1 incremental checker (oracle/, as it stands) on the first ncols columns of the
    workload: the fair analogue of the paper's scalar-integer reference."""
    import oracle
    oracle.build()
    t0 = time.perf_counter()
    oracle.eval_incremental(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, ncols)
    return w.t * ncols, time.perf_counter() - t0


def oracle_sample(w, ncols: int, seed: int = 0):
    """Time the direct oracle (as it stands) on ncols sampled columns of the workload."""
    import oracle
    oracle.build()
    rng = np.random.default_rng(seed)
    ks = np.sort(rng.choice(w.T, size=min(ncols, w.T), replace=False)).astype(np.uint64)
    t0 = time.perf_counter()
    oracle.eval_workload(w, ks=ks)
    dt = time.perf_counter() - t0
    return w.t * len(ks), dt, ks


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    cores = host_cores()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    ncols = cores                                   # one sampled column per core per step
    times = []
    tp = 0
    for i in range(args.warmup + args.steps):
        n_tp, dt, _ = oracle_sample(w, ncols, seed=i)
        if i >= args.warmup:
            times.append(dt)
            tp = n_tp
    ms = 1e3 * statistics.mean(times)
    value = tp / (ms * 1e-3)
    sample = f"{w.name}: all {w.t} terms x {ncols} sampled columns of T={w.T} per step (direct oracle)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": workload_config(w),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(w):
    """The workload only (identical in both arms); implementation details go to impl_config."""
    return {"workload": w.name, "t": w.t, "n": w.n, "T": w.T, "j0": w.j0, "p": w.p,
            "term_points_per_step": w.t * w.T,
            "l2": ("inputs larger than L2 (126 MB): the tensor-core step streams the handle's 10 GB of "
                   "giant-step planes (1 KB per term; 0.5 KB of baby-step planes in the plain form) + "
                   "0.8 GB of per-term records per launch (config 5); the scalar step reads c, m, w "
                   "(3 x 8 B x t_padded)")}


def impl_config(info):
    return {"kernel": "k_tc" if info.get("uses_tc") else "k_step", "scalar_core": info["path"], "R": info["R"],
            "warps": info["warps"], "t_padded": info["t_padded"], "n_slots": info["n_slots"], "G": info.get("G"),
            "tc_pieces": info.get("tc_pieces")}


# ---------------------------------------------------------------- GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-cols", type=int, default=0, help="oracle sample columns (0 = 4 x cores)")
    ap.add_argument("--sustain-s", type=float, default=3.0,
                    help="also run the device step back to back for this many seconds (power-capped "
                         "figure, reported as 'sustained'; 0 skips it)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    import synth
    t0 = time.perf_counter()
    w = synth.gen_config(args.config)
    log(f"[rank {rank}] generated {w.name}: t={w.t} n={w.n} T={w.T} in {time.perf_counter() - t0:.1f}s")

    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2004_11571_b200 as pe
    from paper_2004_11571_b200.dist import ShardedEval, TermShardedEval, bucket_keys, term_partition

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product path has no CPU fallback)")
    torch.cuda.set_device(local_rank)
    if world > 1:
        # communicator set-up lines (nranks, NVLS/NVLink transport) on stderr, for the run's log;
        # stdout stays the single JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- multi-GPU decomposition: the tensor-core path works in whole 8192-point chunks, so with
    # N > 1 ranks shard bucket-contiguous TERM ranges (each rank: all T points of ~t/N terms,
    # P2P row gather, boundary buckets summed mod p by pe_rows_addmod) -- measured 6.5x vs 1.55x
    # for point ranges at 8 ranks; the scalar path shards the point range.
    probe = pe.Context(w.p, w.coeffs[:1], w.exps[:1], w.alpha, n=w.n)
    term_shard = world > 1 and probe.uses_tc(w.T)
    probe.close()
    if term_shard:
        order, bounds = term_partition(w.exps, world)
        mine = np.sort(order[bounds[rank]:bounds[rank + 1]])
        w_c, w_e = np.ascontiguousarray(w.coeffs[mine]), np.ascontiguousarray(w.exps[mine])
    else:
        w_c, w_e = w.coeffs, w.exps

    # ---- handle (pe_create) -- outside the device-timed region
    t0 = time.perf_counter()
    ctx = pe.Context(w.p, w_c, w_e, w.alpha, n=w.n)
    torch.cuda.synchronize()
    create_s = time.perf_counter() - t0
    info = ctx.info()
    info["G"] = ctx.G
    if term_shard:
        sh = TermShardedEval(bucket_keys(w.exps)[order], bounds, w.T, w.p, dev)
        # one launch per rank, then the gather: splitting a rank's rows into two launches to hide
        # the gather under the second (TermShardedEval.run_blocks) costs more than the 0.13 ms it
        # hides at 8 ranks (scripts/partition_probe.py: 6.36x vs 6.56x predicted)
        info["G"] = sh.G
        local_tp = w_c.size * w.T
        info["uses_tc"] = ctx.uses_tc(w.T)

        def step():
            return sh.run(lambda out: ctx.eval_device(w.j0, w.T, out.data_ptr(), w.T, stream.cuda_stream))
    else:
        sh = ShardedEval(ctx.G, w.T, dev)
        local_tp = w.t * sh.cnt
        info["uses_tc"] = ctx.uses_tc(sh.cnt)

        def eval_local(j_first, cnt, out):
            ctx.eval_device(j_first, cnt, out.data_ptr(), out.shape[1], stream.cuda_stream)

        def step():
            return sh.run(eval_local, w.j0)

    # ---- end-to-end: host inputs -> host result through the C ABI, every step
    def run_e2e():
        e2e = None
        if not args.no_e2e:
            pin = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64) if a.dtype == np.uint64
                                             else np.ascontiguousarray(a).view(np.int32)).pin_memory()
            h_c, h_e, h_a = pin(w_c), pin(w_e), pin(w.alpha)          # this rank's terms (all for N = 1)
            G_all = sh.G if term_shard else ctx.G
            h_out = torch.empty((G_all, w.T), dtype=torch.int64).pin_memory() if sh.is_root else None
            L = pe.lib()
            import ctypes

            def create_h(compact=False):
                if compact:
                    h = L.pe_create_compact(w.p, w.t, w.n, ctypes.c_void_p(h_c.data_ptr()),
                                            ctypes.c_void_p(h_e8.data_ptr()), ctypes.c_void_p(h_a.data_ptr()), None)
                else:
                    h = L.pe_create(w.p, w_c.size, w.n, ctypes.c_void_p(h_c.data_ptr()),
                                    ctypes.c_void_p(h_e.data_ptr()), ctypes.c_void_p(h_a.data_ptr()))
                if not h:
                    raise pe.PEError(L.pe_last_error(), "pe_create")
                return h

            def eval_h(h):
                try:
                    if world == 1:
                        rc = L.pe_eval(h, w.j0, w.T, ctypes.c_void_p(h_out.data_ptr()))
                        if rc:
                            raise pe.PEError(rc, "pe_eval")
                    elif term_shard:
                        def ev_rows(out):
                            rc = L.pe_eval_device(h, w.j0, w.T, ctypes.c_void_p(out.data_ptr()), w.T,
                                                  ctypes.c_void_p(stream.cuda_stream))
                            if rc:
                                raise pe.PEError(rc, "pe_eval_device")
                        res = sh.run(ev_rows)
                        if sh.is_root:
                            h_out.copy_(res)
                        torch.cuda.synchronize()
                    else:
                        def ev(j_first, cnt, out):
                            rc = L.pe_eval_device(h, j_first, cnt, ctypes.c_void_p(out.data_ptr()), out.shape[1],
                                                  ctypes.c_void_p(stream.cuda_stream))
                            if rc:
                                raise pe.PEError(rc, "pe_eval_device")
                        res = sh.run(ev, w.j0)
                        if sh.is_root:
                            h_out.copy_(res)
                        torch.cuda.synchronize()
                finally:
                    L.pe_destroy(h)

            nrep = max(3, min(args.steps, 5))

            def serial(compact=False):
                # latency: one polynomial at a time, create -> eval -> result on the host
                for _ in range(2):
                    eval_h(create_h(compact))
                ts = []
                for _ in range(nrep):
                    barrier()
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    eval_h(create_h(compact))
                    torch.cuda.synchronize()
                    ts.append(max_over_ranks(time.perf_counter() - t0))
                return statistics.median(ts)

            h_e8 = None
            if world == 1 and int(w.exps.max()) < 256:
                h_e8 = torch.from_numpy(np.ascontiguousarray(w.exps.astype(np.uint8))).pin_memory()
            e2e_s = serial()
            # the same through pe_create_compact (uint8 exponents: 120 MB instead of 480 MB over PCIe;
            # every config's degrees are < 256), single GPU only
            e2e_c = None
            if h_e8 is not None:
                ec = serial(True)
                e2e_c = {"value": w.t * w.T / ec, "unit": UNIT, "ms_per_step": 1e3 * ec,
                         "h2d_bytes_per_step": w.coeffs.nbytes + h_e8.numel() + w.alpha.nbytes,
                         "d2h_bytes_per_step": ctx.G * w.T * 8,
                         "includes": "pe_create_compact (uint8 exponents) + pe_eval, host wall clock"}
            # the host result of the last e2e polynomial must equal the device-timed path's output
            ref = step()
            torch.cuda.synchronize()
            e2e_ok = bool(torch.equal(ref.cpu(), h_out)) if sh.is_root else None
            if sh.is_root and not e2e_ok:
                raise SystemExit("bench.py: e2e host result differs from the device path's output")
            h2d = (w.coeffs.nbytes + w.exps.nbytes + w.alpha.nbytes * world if term_shard
                   else (w.coeffs.nbytes + w.exps.nbytes + w.alpha.nbytes) * world)
            e2e = {"value": w.t * w.T / e2e_s, "unit": UNIT, "ms_per_step": 1e3 * e2e_s,
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": G_all * w.T * 8,
                   "includes": "one polynomial at a time: pe_create (H2D + sort + plan + K1) + eval + gather "
                               "+ D2H, host wall clock, max over ranks",
                   "matches_device_result": e2e_ok,
                   "compact_exponents": e2e_c}

        return e2e


    # ---- device-timed region (clock samples from the warm-up on: nvidia-smi starts slowly)
    with ClockSampler(local_rank) as clk:
        t_load0 = time.time()
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        ctx.kernel_stats()                      # drop anything recorded so far
        barrier()
        torch.cuda.synchronize()
        ctx.set_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        t_load1 = time.time()
        time.sleep(0.15)                        # let the sampler flush its last line
    barrier()
    ctx.set_timing(False)
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    ks = ctx.kernel_stats()
    value = w.t * w.T / (ms * 1e-3)
    clocks = clk.summary(t_load0, t_load1)

    # ---- optional sustained leg: back-to-back steps for >= args.sustain_s seconds (power-capped clock)
    sustained = None
    if args.sustain_s > 0:
        n_s = max(1, int(args.sustain_s * 1e3 / ms))
        with ClockSampler(local_rank) as clk2:
            barrier()
            torch.cuda.synchronize()
            ts0 = time.time()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(n_s):
                step()
            f1.record(stream)
            torch.cuda.synchronize()
            ts1 = time.time()
            time.sleep(0.15)
        ms_s = max_over_ranks(f0.elapsed_time(f1) / n_s)
        sustained = {"steps": n_s, "seconds": n_s * ms_s / 1e3, "ms_per_step": ms_s,
                     "value": w.t * w.T / (ms_s * 1e-3), "clocks": clk2.summary(ts0, ts1)}

    # ---- roofline of the dominant kernel (k_tc on the tensor-core path, else k_step)
    pk, pk_kind = peaks()
    n_launch = max(ks["step_launches"], 1)                                 # passes x steps (rank 0)
    step_ms = ks["step_ms"] / n_launch                                     # mean launch time
    launches_tp = ks["term_points"] / n_launch                             # padded term-points / launch
    algo_tp = local_tp * args.steps / n_launch if local_tp else 0         # algorithmic term-points / launch
    tp_rate = algo_tp / (step_ms * 1e-3) if step_ms else 0.0
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    imad_peak = N_SM * sm_mhz * 1e6 * IMAD_LANES_PER_CLK_SM / IMAD_SLOTS_PER_TP
    use_tc = info["uses_tc"]
    if use_tc:
        # 64 exact byte-pair multiply-accumulates per term-point: 128 int8 ops
        ops = algo_tp * OPS_PER_TP_TC
        achieved = ops / (step_ms * 1e-3)
        peak = pk.get("bf16_tflops", 1590.0) * 1e12 * 2            # int8 dense = 2 x bf16 (guide nominal)
        mma = {n: pe.bench_mma(n) for n in (64, 128)}                # same-run tcgen05 i8 issue rate
        traffic, traffic_src = ncu_traffic("ktc")
        roof = {"bound": "tensor", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "k_tc (tcgen05.mma kind::i8 M=128 N=64..256 K=32, u8 x u8 -> s32 in TMEM)",
                "peak_basis": (f"int8 dense tensor ops = 2 x {pk_kind} bf16_tflops "
                               f"{pk.get('bf16_tflops', 1590.0):.1f} (guide nominal ratio 4.5/2.25 PFLOP/s); "
                               f"sustained basis 2 x {pk.get('bf16_tflops_sustained', 1375.5):.1f}"),
                "frac_of_sustained": achieved / (2e12 * pk.get("bf16_tflops_sustained", 1375.5)),
                "mma_n128_ceiling": mma[128] / 1e12, "frac_of_mma_n128_ceiling": achieved / mma[128],
                "mma_n64_ceiling": mma[64] / 1e12,
                "term_points_per_s": tp_rate / 1e12,
                "speedup_vs_imad_mulmod_roofline": tp_rate / imad_peak,
                "imad_mulmod_roofline": imad_peak / 1e12,
                "step_ms": step_ms, "fixup_ms": ks["fixup_ms"] / n_launch,
                "padded_term_points_per_launch": launches_tp, "term_points_per_launch": algo_tp,
                "int8_ops_per_launch": ops, "tc_pieces": info["tc_pieces"],
                "algorithmic_bytes_per_launch": 16 * w_c.size + 8 * ctx.G * w.T}
        gpu_launches = 3 * ks["step_launches"]       # k_tc_seed + k_tc + k_fixup per pass (rank 0)
    else:
        achieved = tp_rate
        peak = imad_peak
        # register-resident ceiling of the same step (K5, no memory / reduction), measured now
        k5 = None
        try:
            k5_ms, k5_steps, _ = pe.bench_core(pe.CORE_SHOUP4 if info["path"] == "int" else pe.CORE_FP64,
                                               w.p, 8, N_SM * 2, 256, 4096)
            k5 = k5_steps / (k5_ms * 1e-3)
        except pe.PEError:
            pass
        traffic, traffic_src = ncu_traffic("kstep") if info["path"] == "int" else (None, None)
        roof = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tterm-pt/s",
                "frac": achieved / peak if peak else None,
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": f"k_step<{info['path']},R={info['R']}>",
                "peak_basis": (f"IMAD-pipe model (DESIGN.md Roofline): {N_SM} SMs x {sm_mhz:.0f} MHz ({pk_kind} "
                               f"sm_max_mhz) x {IMAD_LANES_PER_CLK_SM} IMAD lanes/clk/SM / {IMAD_SLOTS_PER_TP} "
                               "IMAD slots per 64-bit Shoup mulmod (4 low x 1 + 5 full-width x 2; measured "
                               "IMAD 64, IMAD.HI 32 lanes/clk/SM, profiles/r01_pipe_bench.jsonl)"),
                "frac_at_run_clock": (achieved / (peak * clocks["sm_mhz"] / sm_mhz)
                                      if clocks.get("sm_mhz") else None),
                "k5_register_resident_ceiling": k5 / 1e12 if k5 else None,
                "frac_of_k5_ceiling": achieved / k5 if k5 else None,
                "step_ms": step_ms, "fixup_ms": ks["fixup_ms"] / n_launch,
                "padded_term_points_per_launch": launches_tp, "term_points_per_launch": algo_tp,
                "algorithmic_bytes_per_launch": 16 * w.t + 8 * ctx.G * sh.cnt}
        gpu_launches = 2 * ks["step_launches"]       # k_step + k_fixup per pass (rank 0)

    e2e = run_e2e()

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if not args.no_cpu and rank == 0 and world == 1:
        cores = host_cores()
        os.environ.setdefault("OMP_NUM_THREADS", str(cores))
        ncols = args.cpu_cols or 4 * cores
        n_tp, dt, _ = oracle_sample(w, ncols)
        inc_cols = max(1, args.cpu_cols or 64)
        i_tp, i_dt = incremental_sample(w, inc_cols)
        cpu = {"value": n_tp / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
               "extrapolated_full_config_s": w.t * w.T / (n_tp / dt),
               "sample": f"{w.name}: all {w.t} terms x {ncols} random columns of T={w.T} "
                         f"(direct definition, OpenMP over columns), {dt:.1f} s",
               "incremental": {"value": i_tp / i_dt, "unit": UNIT, "cores": cores,
                               "extrapolated_full_config_s": w.t * w.T / (i_tp / i_dt),
                               "sample": f"Alg. 1 checker (oracle incr_eval, OpenMP over rows): all {w.t} terms x "
                                         f"the first {inc_cols} columns, {i_dt:.1f} s"}}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": workload_config(w), "impl_config": impl_config(info), "roofline": roof,
                "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": gpu_launches, "clocks": clocks, "sustained": sustained,
                "create_s": create_s,
                "parallelism": ("single GPU (no collective)" if world == 1 else
                                f"bucket-contiguous term ranges x{world}, NCCL P2P row gather + pe_rows_addmod"
                                if term_shard else f"point-range shards x{world}, NCCL gather + pe_unshard_columns")}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
