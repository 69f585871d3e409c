"""Summarise an ncu report (or a launch-list CSV) into a small markdown table.

    python profiles/summarize_ncu.py gpurun_out/prof.ncu-rep > profiles/rNN/x.md
    python profiles/summarize_ncu.py --launches gpurun_out/launches.csv [--last N]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active", "imma active %"),
    ("sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed", "int8 ops % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize_rep(rep):
    hdr, units, rows = raw_rows(rep)
    cols = ["kernel", "grid"] + [name for _, name in KEYS]
    print("| " + " | ".join(cols) + " |")
    print("|" + "---|" * len(cols))
    for r in rows:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        vals = [d.get("Kernel Name", "")[:48], d.get("Grid Size", "")]
        for key, _ in KEYS:
            v = d.get(key, "")
            unit = u.get(key, "")
            vals.append(f"{v} {unit}".strip())
        print("| " + " | ".join(vals) + " |")


def summarize_launches(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr = None
    out = []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["ID"], d["Kernel Name"], d["Grid Size"], float(d["Metric Value"]), d["Metric Unit"]))
    if last:
        out = out[-last:]
    total = sum(o[3] for o in out)
    print("| id | kernel | grid | time | share |")
    print("|---|---|---|---|---|")
    for o in out:
        print(f"| {o[0]} | {o[1][:70]} | {o[2]} | {o[3]:.0f} {o[4]} | {100 * o[3] / total:.1f}% |")
    print(f"\ntotal {total:.0f} over {len(out)} launches")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        last = int(sys.argv[sys.argv.index("--last") + 1]) if "--last" in sys.argv else None
        summarize_launches(sys.argv[2], last)
    else:
        summarize_rep(sys.argv[1])
