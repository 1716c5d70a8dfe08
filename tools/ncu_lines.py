"""Per-source-line instruction counts / stall samples of one kernel of an ncu
report, by matching the report's SASS (in order) to `nvdisasm -g` line info of
the same cubin.  Usage: ncu_lines.py REPORT KERNEL_INDEX OBJ MANGLED_SUBSTR [N]"""
import re
import subprocess
import sys
import tempfile
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).parent))
from ncu_sass_top import load, num  # noqa: E402


def disasm_lines(obj, func_sub):
    tmp = Path(tempfile.mkdtemp())
    subprocess.run(["cuobjdump", "-xelf", "all", str(Path(obj).resolve())], cwd=tmp, capture_output=True)
    out = ""
    for cubin in sorted(tmp.glob("*.cubin")):  # the object holding the function
        out = subprocess.run(["nvdisasm", "-g", "-c", str(cubin)], capture_output=True, text=True).stdout
        if func_sub in out:
            break
    lines, cur, infn = [], None, False
    for l in out.splitlines():
        if l.startswith(".text.") or re.match(r"^\s*\.section\s+\.text\.", l):
            infn = func_sub in l
            continue
        m = re.search(r'//## File ".*", line (\d+)', l)
        if m:
            cur = int(m.group(1))
            continue
        if infn and re.match(r"\s+/\*[0-9a-f]{4,}\*/", l):
            lines.append(cur)
    return lines


def main(rep, which, obj, func_sub, n=40):
    rows = load(rep, which)
    lines = disasm_lines(obj, func_sub)
    print(f"{len(rows)} sass rows in report, {len(lines)} in cubin")
    ins, smp = defaultdict(float), defaultdict(float)
    for r, ln in zip(rows, lines):
        ins[ln] += num(r["Instructions Executed"])
        smp[ln] += num(r["Warp Stall Sampling (All Samples)"])
    ti, ts = sum(ins.values()), sum(smp.values())
    src = Path(__file__).resolve().parents[1] / "paper_1604_04026_b200/csrc/solve_fast.cu"
    text = src.read_text().splitlines()
    key = smp if "--samples" in sys.argv else ins
    for ln in sorted(ins, key=lambda k: -key[k])[:n]:
        code = text[ln - 1].strip()[:70] if ln else "?"
        print(f"  line {ln}: inst {100 * ins[ln] / ti:5.1f}%  samples {100 * smp[ln] / ts:5.1f}%  {code}")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    main(args[0], int(args[1]), args[2], args[3], int(args[4]) if len(args) > 4 else 40)
