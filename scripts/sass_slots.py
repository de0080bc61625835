"""Count IMAD-pipe (fmaheavy) slots per term-point in the hot loop of a compiled kernel.

    python scripts/sass_slots.py <lib.so|cubin> <mangled-kernel-substring> [term_points_per_iter]

Cost model (measured, profiles/r01_pipe_bench.jsonl): IMAD / IMAD.MOV / IMAD.IADD / IMAD.X /
IMAD.SHL = 1 slot, IMAD.WIDE / IMAD.HI = 2 slots (64 slots/clk/SM).  The hot loop is the
backward branch whose body holds the most IMAD.HI + IMAD.WIDE + DFMA.
"""
import collections
import re
import subprocess
import sys

COST = {"IMAD": 1, "IMAD.MOV.U32": 1, "IMAD.MOV": 1, "IMAD.IADD": 1, "IMAD.X": 1, "IMAD.SHL.U32": 1,
        "IMAD.WIDE.U32": 2, "IMAD.WIDE": 2, "IMAD.HI.U32": 2, "IMAD.WIDE.U32.X": 2, "IMAD.HI.U32.X": 2}


def hot_loop(sass: str):
    ins = []
    for l in sass.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d\s*,\s*)?(0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            tgt = int(m.group(1), 16)
            body = [y for x, y in ins if tgt <= x <= a]
            key = sum(("IMAD.HI" in y) or ("IMAD.WIDE" in y) or ("DFMA" in y) for y in body)
            if best is None or key > best[0]:
                best = (key, body)
    return best[1] if best else []


def opcode(t):
    t = re.sub(r"^@!?U?P\w+\s+", "", t)
    return t.split()[0]


def main():
    lib, name = sys.argv[1], sys.argv[2]
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", sass)
    f = next(x for x in funcs if x.split("\n")[0].strip().find(name) >= 0)
    body = hot_loop(f)
    c = collections.Counter(opcode(t) for t in body)
    n_hi = c["IMAD.HI.U32"]
    tp = float(sys.argv[3]) if len(sys.argv) > 3 else None
    slots = sum(COST.get(k, 0) * v for k, v in c.items())
    print(f"{f.split(chr(10))[0].strip()}: {len(body)} instr, IMAD slots {slots}")
    if tp:
        print(f"  per term-point: instr {len(body) / tp:.2f}, IMAD slots {slots / tp:.2f}")
    for k, v in c.most_common(16):
        print(f"  {v:6d} {k}" + (f"  ({v / tp:.2f}/tp)" if tp else ""))


if __name__ == "__main__":
    main()
