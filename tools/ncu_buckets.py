"""Per-launch table (markdown) of an ncu report of all solver launches:
duration, DRAM traffic and achieved GB/s, achieved occupancy, issue activity,
FP64 pipe, shared-memory throughput and bank conflicts, top warp-stall
reasons.  Usage: ncu_buckets.py REPORT|RAW_CSV"""
import csv
import io
import re
import subprocess
import sys

COLS = {
    "gpu__time_duration.sum": "dur",
    "dram__bytes.sum.per_second": "bw",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ",
    "sm__inst_executed.avg.pct_of_peak_sustained_elapsed": "issue",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed": "fp64",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "regs",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "conf",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "wavef",
    "dram__bytes_read.sum": "dread",
    "dram__bytes_write.sum": "dwrite",
}
STALL = "smsp__average_warps_issue_stalled_"
STALL_END = "_per_issue_active.ratio"


def to_num(v, unit):
    v = float(v.replace(",", ""))
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "byte/second": 1e-9, "Kbyte/second": 1e-6, "Mbyte/second": 1e-3, "Gbyte/second": 1.0,
             "Tbyte/second": 1e3, "Gbyte/s": 1.0, "Tbyte/s": 1e3, "Mbyte/s": 1e-3}
    return v * scale.get(unit, 1.0)


def main(path):
    if path.endswith(".csv"):  # an exported raw page (ncu -i REP --page raw --csv)
        raw = open(path).read()
    else:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    print("| # | kernel | grid | regs | ms | DRAM GB | DRAM GB/s | occupancy % | issue % | FP64 % | SMEM % | "
          "bank conflicts / wavefronts | top stalls (warps per issue) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for q, r in enumerate(data):
        get = {}
        for i, h in enumerate(hdr):
            if h in COLS:
                get[COLS[h]] = to_num(r[i], units[i]) if r[i] else 0.0
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith(STALL) and h.endswith(STALL_END) and r[i] and "selected" not in h:
                stalls.append((float(r[i].replace(",", "")), h[len(STALL):-len(STALL_END)]))
        stalls.sort(reverse=True)
        name = re.sub(r"\(klnmf_solve_args_t.*", "", r[ki]).replace("klnmf::<unnamed>::", "").replace("void ", "")
        name = name.replace("(int)", "")
        ms = get.get("dur", 0.0)
        top = ", ".join(f"{n} {v:.2f}" for v, n in stalls[:3])
        dram = (get.get("dread", 0.0) + get.get("dwrite", 0.0)) / 1e9
        conf = get.get("conf", 0.0) / max(get.get("wavef", 0.0), 1.0)
        print(f"| {q} | {name} | {get.get('grid', 0):.0f} | {get.get('regs', 0):.0f} | {ms:.3f} | {dram:.3f} | "
              f"{get.get('bw', 0):.0f} | {get.get('occ', 0):.0f} | {get.get('issue', 0):.0f} | "
              f"{get.get('fp64', 0):.0f} | {get.get('smem', 0):.0f} | {conf:.2f} | {top} |")


if __name__ == "__main__":
    main(sys.argv[1])
