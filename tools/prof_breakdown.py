"""Per-phase instruction / stall breakdown of k_warp from an ncu report.
python tools/prof_breakdown.py REP [kernel-prefix]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1]
pref = sys.argv[2] if len(sys.argv) > 2 else "_ZN2xb6k_warpILi1ELb0ELb0ELi4E"
out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_lines.py"), rep, pref, "-", "100000"],
                     capture_output=True, text=True, env=dict(os.environ, XB_NCU_KERNEL="k_warp")).stdout
rows = []
for ln in out.splitlines()[1:]:
    p = ln.split()
    f, l = p[0].rsplit(":", 1)
    rows.append((f, int(l), float(p[1]), float(p[2]), float(p[3])))


def agg(name, pred):
    s = sum(r[2] for r in rows if pred(r))
    i = sum(r[3] for r in rows if pred(r))
    thr = sum(r[3] * r[4] for r in rows if pred(r)) / max(i, 1e-9)
    print(f"{name:28s} stall {s:6.1f}%  inst {i:6.1f}%  thr/warp {thr:5.1f}")


src = open(os.path.join(ROOT, "paper_2009_03076_b200/csrc/render.cu")).read().splitlines()
msrc = open(os.path.join(ROOT, "paper_2009_03076_b200/csrc/march.cuh")).read().splitlines()


def find(lines, pat, start=0):
    for i, l in enumerate(lines):
        if i >= start and pat in l:
            return i + 1
    return 10 ** 9


kw = find(src, "k_warp(const __grid_constant__")
c0 = find(src, "// ================= one chunk", kw)
sc = find(src, "inclusive scan of the front-to-back", kw)
tr = find(src, "// ================= traversal", kw)
co = find(src, "// ---- consume leading leaves", kw)
ex = find(src, "// ---- expansion step", kw)
en = find(src, "if (lane == 0) {", co)
R = lambda x, y: (lambda r: r[0] == "render.cu" and x <= r[1] < y)
agg("ray setup", R(kw, c0))
agg("chunk map + eval", R(c0, sc))
agg("scan + queue drop", R(sc, tr))
agg("list / frontier refill", R(tr, ex))
agg("expand", R(ex, co))
agg("consume leaves", R(co, en))
agg("pixel write", R(en, en + 40))
agg("render.cu helpers", lambda r: r[0] == "render.cu" and not (kw <= r[1] < en + 40))
g0 = find(msrc, "void gather_shade(")
g1 = find(msrc, "double shade_factor_f")
agg("gather_shade", lambda r: r[0] == "march.cuh" and g0 <= r[1] < g1)
agg("march.cuh other", lambda r: r[0] == "march.cuh" and not (g0 <= r[1] < g1))
agg("intrinsics", lambda r: "intrinsics" in r[0])
agg("other headers", lambda r: r[0] not in ("render.cu", "march.cuh") and "intrinsics" not in r[0])
