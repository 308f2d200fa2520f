"""Summarise an ncu report (and an optional launch list) into a short text
file for profiles/.  Usage: python tools/ncu_summary.py REP.ncu-rep [launches.csv] > out.txt"""
import csv
import subprocess
import sys
from collections import defaultdict


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def main():
    rep = sys.argv[1]
    rows = ncu_csv(rep, "details")
    h = rows[0]
    k_i, m_i, u_i, v_i = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    id_i = h.index("ID")
    keep = ("Duration", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Achieved Occupancy", "Theoretical Occupancy", "Avg. Active Threads Per Warp",
            "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Executed Instructions",
            "Branch Efficiency", "Grid Size", "Block Size", "Stack Size")
    print(f"# ncu --set full summary: {rep}")
    raw = ncu_csv(rep, "raw")
    rh = raw[0]
    ids = []
    for r in rows[1:]:
        if r[id_i] not in ids:
            ids.append(r[id_i])
    for kid in ids:
        kr = [r for r in rows[1:] if r[id_i] == kid]
        print(f"kernel: {kr[0][k_i]}")
        for r in kr:
            if r[m_i] in keep:
                print(f"  {r[m_i]:40s} {r[v_i]:>16s} {r[u_i]}")
        rr = [x for x in raw[2:] if x[rh.index("ID")] == kid]
        if not rr:
            continue
        d = dict(zip(rh, rr[0]))
        u = dict(zip(rh, raw[1]))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
                  "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
                  "smsp__thread_inst_executed.sum"):
            if k in d:
                print(f"  {k:60s} {d[k]:>16s} {u.get(k, '')}")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("  warp stall samples (share):")
        for v, k in sorted(st, reverse=True)[:8]:
            print(f"    {k:28s} {100 * v / tot:5.1f} %")
    if len(sys.argv) > 2:
        rows = list(csv.reader(open(sys.argv[2])))
        hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        h = rows[hi]
        ki, vi = h.index("Kernel Name"), h.index("Metric Value")
        t, c = defaultdict(float), defaultdict(int)
        for r in rows[hi + 1:]:
            try:
                t[r[ki][:70]] += float(r[vi].replace(",", ""))
                c[r[ki][:70]] += 1
            except (ValueError, IndexError):
                pass
        tot = sum(t.values())
        print(f"# launch list {sys.argv[2]} (gpu__time_duration.sum, cold/serialised; compare shares)")
        for k, v in sorted(t.items(), key=lambda x: -x[1])[:12]:
            print(f"  {v / 1e6:9.3f} ms {100 * v / tot:5.1f}%  n={c[k]:4d}  {k}")


if __name__ == "__main__":
    main()
