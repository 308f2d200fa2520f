"""Attribute an ncu SASS source page to CUDA source lines.

  python tools/sass_lines.py REP.ncu-rep KERNEL_MANGLED_PREFIX [cubin] [top]

Maps each SASS offset to the innermost `//## File ..., line N` comment of
`nvdisasm -g` on the cubin (default: render.sm_100a.cubin extracted from
libexabricks.so), then sums ncu's stall samples and executed instructions per
(file, line)."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_csv(rep, kfilter=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    if kfilter:
        cmd += ["-k", "regex:" + kfilter]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    body = []
    for r in rows[2:]:  # first kernel block only
        if r and r[0] == "Kernel Name":
            break
        if r and r[0].startswith("0x"):
            body.append(r)
    return hdr, body


def line_map(cubin, prefix):
    out = subprocess.run(["nvdisasm", "-g", cubin], capture_output=True, text=True).stdout
    m, cur, inside = {}, None, False
    for ln in out.splitlines():
        if ln.startswith(".text."):
            inside = ln[len(".text."):].startswith(prefix)
            continue
        if not inside:
            continue
        g = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if g:
            cur = (os.path.basename(g.group(1)), int(g.group(2)))
            continue
        g = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
        if g:
            m[int(g.group(1), 16)] = (cur, g.group(2).strip())
    return m


def main():
    rep, prefix = sys.argv[1], sys.argv[2]
    cubin = sys.argv[3] if len(sys.argv) > 3 and sys.argv[3] != "-" else None
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    if cubin is None:
        d = tempfile.mkdtemp()
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_2009_03076_b200", "libexabricks.so")],
                       cwd=d, capture_output=True)
        cubin = os.path.join(d, "render.sm_100a.cubin")
    lm = line_map(cubin, prefix)
    kf = os.environ.get("XB_NCU_KERNEL")  # e.g. k_warp when the report holds several kernels
    hdr, rows = sass_csv(rep, kf)
    ia, ist, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index(
        "Instructions Executed")
    ith = hdr.index("Thread Instructions Executed")
    base = int(rows[0][ia], 16)
    agg = defaultdict(lambda: [0, 0, 0])
    tot = [0, 0, 0]
    for r in rows:
        off = int(r[ia], 16) - base
        key = lm.get(off, (("?", 0), ""))[0] or ("?", 0)
        v = [int(r[ist] or 0), int(r[iex] or 0), int(r[ith] or 0)]
        for i in range(3):
            agg[key][i] += v[i]
            tot[i] += v[i]
    print(f"{'file:line':32s} {'stall%':>7s} {'inst%':>7s} {'thr/warp':>8s}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{k[0] + ':' + str(k[1]):32s} {100 * v[0] / max(tot[0], 1):7.2f} {100 * v[1] / max(tot[1], 1):7.2f} "
              f"{v[2] / max(v[1], 1):8.1f}")


if __name__ == "__main__":
    main()
