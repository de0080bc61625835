"""Summarise an ncu --set full report of one kernel launch: duration, pipe utilisation, tensor
activity, DRAM traffic, issue activity, and the top warp-stall sites (SASS).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json] [--top 25]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_active.avg": "sm_cycles_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "issue_active_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "fmaheavy_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed": "alu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_elapsed": "lsu_pct",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.sum": "utcimma_ops",
    "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.per_cycle_elapsed": "utcimma_ops_per_clk_sm",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                out[KEYS[h]] = (float(v.replace(",", "")), u)
            except ValueError:
                out[KEYS[h]] = (v, u)
    return out


def stalls(rep, top):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source", "sass"))))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    st = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = {s: 0 for s in st}
    sites = []
    for r in rows[2:]:
        try:
            n = int(r[ix["# Samples"]] or 0)
        except (ValueError, IndexError):
            continue
        for s in st:
            try:
                tot[s] += int(r[ix[s]] or 0)
            except ValueError:
                pass
        top_reason = max(st, key=lambda s: int(r[ix[s]]) if r[ix[s]].isdigit() else 0)
        sites.append((n, r[ix["Address"]][-5:], r[ix["Instructions Executed"]], r[ix["Source"]][:70], top_reason))
    sites.sort(key=lambda x: -x[0])
    return tot, sites[:top]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 25
    m = raw(rep)
    for k, (v, u) in m.items():
        print(f"{k:28s} {v} {u}")
    tot, sites = stalls(rep, top)
    n = sum(tot.values()) or 1
    print("stall reasons (% of samples):", {k[6:]: round(100 * v / n, 1) for k, v in
                                           sorted(tot.items(), key=lambda x: -x[1]) if v})
    for s in sites:
        print(f"{s[0]:8d} {s[1]} exec={s[2]:>10s} {s[4][6:]:14s} {s[3]}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump({"metrics": {k: v for k, (v, _) in m.items()}, "stalls": tot}, f, indent=1)


if __name__ == "__main__":
    main()
