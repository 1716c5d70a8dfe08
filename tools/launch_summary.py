"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
bench.py: the kernels of the last outer iteration (after the last L2 flush),
their cold-cache, serialised durations and their share of that iteration."""
import csv
import re
import sys
from collections import OrderedDict


def short(name):
    m = re.search(r"(solve_\w+?)(?:<([^>]*)>)?\(", name)
    if m:
        return m.group(1) + (f"<{m.group(2).replace('(int)', '')}>" if m.group(2) else "")
    m = re.search(r"(\w+)(?:<.*>)?\(", name)
    return (m.group(1) if m else name)[:40]


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui, gi, bi = (hdr.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit", "Grid Size",
                                                 "Block Size"))
    launches = []
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        v = v / 1e6 if r[ui] == "ns" else (v / 1e3 if r[ui] in ("us", "usecond") else v)
        launches.append((r[ki], r[gi], r[bi], v))
    # the last timed step starts after bench.py's device sleep (spin_kernel)
    # and ends at the next fill (stats reset / L2 flush of what follows:
    # bench.py's serialised instrumented pass)
    last = max(i for i, l in enumerate(launches) if "spin_kernel" in l[0])
    step = []
    for l in launches[last + 1:]:
        if "FillFunctor" in l[0]:
            break
        step.append(l)
    tot = sum(l[3] for l in step)
    agg = OrderedDict()
    for name, grid, block, ms in step:
        k = (short(name), block)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ms
    print(f"launches in the last timed iteration: {len(step)}, serialised sum {tot:.2f} ms")
    print("| kernel | block | launches | ms | share |")
    print("|---|---|---|---|---|")
    for (k, b), (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {b} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
