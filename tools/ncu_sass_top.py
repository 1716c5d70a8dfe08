"""Top SASS instructions of an ncu report by stall samples / excess shared wavefronts."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def load(path, which=0):
    """SASS rows of the which-th kernel of the report."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = out.split('"Kernel Name"')[1:]
    lines = blocks[which].splitlines()
    print("kernel:", lines[0][:120])
    i = next(k for k, l in enumerate(lines) if l.startswith('"Address"'))
    return list(csv.DictReader(io.StringIO("\n".join(lines[i:]))))


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main(path, n=40, which=0):
    rows = load(path, which)
    tot = sum(num(r["Warp Stall Sampling (All Samples)"]) for r in rows)
    print(f"{len(rows)} instructions, {tot:.0f} samples")
    by_op = defaultdict(float)
    by_op_ex = defaultdict(float)
    stall_cols = [c for c in rows[0] if c.startswith("stall_") and "Not Issued" not in c]
    stall_tot = defaultdict(float)
    for r in rows:
        op = r["Source"].split()[0] if r["Source"].split() else "?"
        if op.startswith("@"):
            op = r["Source"].split()[1]
        op = op.split(".")[0]
        by_op[op] += num(r["Warp Stall Sampling (All Samples)"])
        by_op_ex[op] += num(r["Instructions Executed"])
        for c in stall_cols:
            stall_tot[c] += num(r[c])
    print("stalls:", ", ".join(f"{k[6:]}={v / tot:.2f}" for k, v in sorted(stall_tot.items(), key=lambda x: -x[1])[:10]))
    print("by opcode (samples%, warp-inst):")
    for op, s in sorted(by_op.items(), key=lambda x: -x[1])[:25]:
        print(f"  {op:10s} {100 * s / tot:5.1f}%  {by_op_ex[op]:.3g}")
    print("top instructions:")
    rows_s = sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))
    for r in rows_s[:n]:
        top = sorted(((num(r[c]), c[6:]) for c in stall_cols), reverse=True)[:2]
        print(f"  {r['Address'][-5:]} {100 * num(r['Warp Stall Sampling (All Samples)']) / tot:5.2f}% "
              f"ex={num(r['Instructions Executed']):.3g} {r['Source'].strip()[:60]:60s} {top}")
    ex = sorted(rows, key=lambda r: -num(r["L1 Wavefronts Shared Excessive"]))
    print("excess shared wavefronts:")
    for r in ex[:10]:
        if num(r["L1 Wavefronts Shared Excessive"]) > 0:
            print(f"  {r['Address'][-5:]} {num(r['L1 Wavefronts Shared Excessive']):.3g} {r['Source'].strip()[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
