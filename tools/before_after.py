"""k_warp before/after table from two ncu --set full reports:
python tools/before_after.py BEFORE.ncu-rep AFTER.ncu-rep [kernel-regex] > profiles/rNN_kwarp_before_after.md"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration (us)", 1e-3),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)", 1),
    ("sm__inst_issued.avg.pct_of_peak_sustained_active", "issue slots busy (%)", 1),
    ("smsp__inst_executed.sum", "warp instructions (M)", 1e-6),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe (%)", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp", 1),
    ("lts__t_sectors.sum.per_second", "L2 throughput (GB/s, 32-B sectors)", 32.0),
    ("lts__t_sectors.sum", "L2 traffic (MB, 32-B sectors)", 32e-6),
    ("dram__bytes.sum.per_second", "DRAM throughput (GB/s)", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1e-6),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit (%)", 1),
    ("launch__registers_per_thread", "registers / thread", 1),
]


def raw(rep, kre):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kre], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, v, u in zip(hdr, vals, units)}


def conv(v, u, scale, name):
    x = float(v.replace(",", ""))
    u = u.strip()
    if name == "dram__bytes.sum.per_second":  # -> GB/s
        x *= {"byte/s": 1e-9, "Kbyte/s": 1e-6, "Mbyte/s": 1e-3, "Gbyte/s": 1, "Tbyte/s": 1e3}.get(u, 1)
    elif name == "lts__t_sectors.sum.per_second":  # sectors/ns * 32 -> GB/s
        x *= {"sector/ns": 1, "sector/us": 1e-3, "sector/s": 1e-9}.get(u, 1)
    elif name.endswith("bytes_read.sum"):
        x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    elif name == "gpu__time_duration.sum":
        x *= {"ns": 1, "us": 1e3, "ms": 1e6}.get(u, 1)
    return x * scale


def main():
    a, b = sys.argv[1], sys.argv[2]
    kre = sys.argv[3] if len(sys.argv) > 3 else "k_warp"
    ra, rb = raw(a, kre), raw(b, kre)
    print(f"| metric ({kre}) | before: {a.split('/')[-1]} | after: {b.split('/')[-1]} |")
    print("|---|---|---|")
    for m, label, sc in METRICS:
        va = conv(*ra[m], sc, m) if m in ra else float("nan")
        vb = conv(*rb[m], sc, m) if m in rb else float("nan")
        print(f"| {label} | {va:.4g} | {vb:.4g} |")


if __name__ == "__main__":
    main()
