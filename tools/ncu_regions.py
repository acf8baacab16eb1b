"""Stall samples and executed instructions of an ncu --set full capture, by SASS
region (regions cut at synchronisation / tensor-memory / copy instructions) and
by opcode.

    python tools/ncu_regions.py gpurun_out/full_x.ncu-rep [min_pct]
"""
import collections
import csv
import io
import subprocess
import sys

MARKS = ("LDTM", "BAR.SYNC", "BAR.RED", "UTCIMMA", "UTCHMMA", "LDGSTS", "SYNCS.ARRIVE",
         "SYNCS.PHASECHK", "EXIT", "STG", "UBLKCP", "RED.")


def main():
    path = sys.argv[1]
    min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 1.5
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[2:] if len(r) > 5]
    k, ex = ix["Warp Stall Sampling (All Samples)"], ix["Instructions Executed"]
    tot = sum(float(r[k] or 0) for r in data) or 1.0
    print(f"{path}: {tot:.0f} stall samples, {sum(float(r[ex] or 0) for r in data):.4g} warp "
          "instructions")
    prev = 0
    for i, r in enumerate(data):
        src = r[ix["Source"]].strip()
        if any(m in src for m in MARKS):
            s = sum(float(data[j][k] or 0) for j in range(prev, i + 1))
            n = sum(float(data[j][ex] or 0) for j in range(prev, i + 1))
            if s / tot * 100 >= min_pct:
                print(f"  [{prev:5d},{i:5d}] {s / tot * 100:5.1f}% stalls {n:10.3g} inst  {src[:60]}")
            prev = i + 1
    ops, st = collections.Counter(), collections.Counter()
    for r in data:
        src = r[ix["Source"]].strip().split()
        op = src[1] if src and src[0].startswith("@") and len(src) > 1 else (src[0] if src else "")
        op = op.split(".")[0]
        ops[op] += float(r[ex] or 0)
        st[op] += float(r[k] or 0)
    n = sum(ops.values()) or 1.0
    print("  opcodes (% of executed, % of stall samples):",
          ", ".join(f"{o} {c / n * 100:.1f}/{st[o] / tot * 100:.1f}" for o, c in ops.most_common(14)))


if __name__ == "__main__":
    main()
