// march.cuh — device functions of the fused ray-march (paper §4, §5).
//
// Everything here restates the reference's FP64 arithmetic operation for
// operation (R/render.py, R/accel.py, R/sampling.py; R/ =
// /root/reference/pkg/src/amrvol/).  The library is compiled with
// -fmad=false so no multiply-add is contracted, like numba's LLVM code.
//
// Region traversal.  The reference finds every next region with a fresh
// closest-hit BVH query from the root, t_start = t_out + eps
// (R/render.py:394-397, R/accel.py:285-352).  Because regions are disjoint
// axis-aligned boxes, their numeric slab intervals [r_in, r_out) are pairwise
// disjoint (slab t's are monotone in the box bounds under IEEE rounding), so
// the closest-hit answer for t_start is simply the first non-empty interval,
// in r_in order, that is not entirely before t_start.  The ABR build is a k-d
// split, so a front-to-back walk of that k-d tree enumerates regions in
// exactly r_in order; culling uses the same monotone arithmetic, so it never
// drops a region the reference would return.  One walk per ray replaces one
// root-to-leaf descent per region visit.
#pragma once
#include "common.cuh"

namespace xb {

constexpr double kEpsWeight = 1e-12;     // EPS_WEIGHT, R/sampling.py:37

constexpr double kTFar = 1.0e30;
// zero pad around the frame gather's value copy: a brick's unclamped 2x2x2
// window reaches at most nx*(ny+1) + 1 <= 32*33 + 1 values before or after it
constexpr int64_t kGatherPad = 2048;         // _T_FAR, R/render.py:49
constexpr int kKdStack = 64;

// exact power of two for |e| < 1022 (brick cell widths, finest widths)
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(1023 + e) << 52); }

struct Ray {
    double o[3], d[3], inv[3];
};

__device__ __forceinline__ double rho_hash(uint64_t pixel, uint64_t seed) {
    // _rho_hash, R/render.py:226-233
    uint64_t z = pixel ^ seed;
    z = z + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ double restart_t(double t_out) {
    // _restart, R/render.py:257-260
    double e = 1e-7 * t_out;
    return t_out + (e > 1e-7 ? e : 1e-7);
}

// _slab, R/accel.py:254-282, on a half-unit integer box (values * 0.5 exact).
// 1/d is hoisted per ray: the reference recomputes the same rounded quotient.
__device__ __forceinline__ void slab_h(const int32_t* lo_h, const int32_t* hi_h, const Ray& r, double& tmin_o,
                                       double& tmax_o) {
    double tmin = -INFINITY, tmax = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; a++) {
        double lo = (double)lo_h[a] * 0.5, hi = (double)hi_h[a] * 0.5;
        if (r.d[a] == 0.0) {
            if (r.o[a] < lo || r.o[a] >= hi) { tmin_o = INFINITY; tmax_o = -INFINITY; return; }
        } else {
            double t0 = (lo - r.o[a]) * r.inv[a], t1 = (hi - r.o[a]) * r.inv[a];
            if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
            if (t0 > tmin) tmin = t0;
            if (t1 < tmax) tmax = t1;
            if (tmin > tmax) { tmin_o = INFINITY; tmax_o = -INFINITY; return; }
        }
    }
    tmin_o = tmin;
    tmax_o = tmax;
}

// the brick build's split tree (SplitTree, R/bricks.py:45-68), preorder, for
// the cell-location gather (use_celllocation); null when absent
struct TreeView {
    const int32_t *axis, *left, *right, *bstart, *bcount;
    const double *lo, *hi, *mh;  // (n,3) boxes, max half cell width
    int64_t n;
};

struct SceneView {
    TreeView tree;
    const int4* __restrict__ brick_a;
    const uint32_t* __restrict__ brick_m;
    const float* __restrict__ vals;
    // the frame gather's copy of the field: vals with kGatherPad zeros before and after
    const float* __restrict__ gvals;
    const RegionRec* __restrict__ rec;
    const int32_t* __restrict__ rids;
    // frame-gather brick records in region-list order (rb[i] = brick rids[i]):
    // a region's bricks are read without the id hop
    const struct RbRec* __restrict__ rb;
    const KdNode* __restrict__ kd;
    const Kd4Node* __restrict__ kd4;
    int32_t root_lo[3], root_hi[3];
    int64_t n_kd, n_kd4;
};

// ---------------------------------------------------------------------------
// ordered k-d walk (see header comment)

struct KdWalk {
    int node;          // current node, -1: pop next
    double tn, tf;     // every region below `node` has tn <= r_in, r_out <= tf
    int sp;
    int st_node[kKdStack];
    float st_tn[kKdStack], st_tf[kKdStack];  // conservative (tn rounded down, tf up)
};

__device__ __forceinline__ void kd_begin(const SceneView& S, const Ray& r, KdWalk& w) {
    double a, b;
    slab_h(S.root_lo, S.root_hi, r, a, b);
    w.sp = 0;
    if (S.n_kd == 0 || !(a <= b)) { w.node = -2; return; }  // ray misses every region
    w.node = 0;
    w.tn = a;
    w.tf = b;
}

// Next region whose interval is non-empty after clipping to [t, tmax] —
// exactly `_bvh_next_hit(t, tmax)` over the regions with flags set.
__device__ __forceinline__ bool kd_next(const SceneView& S, const uint8_t* __restrict__ flags, const Ray& r, KdWalk& w,
                                        double t, double tmax, int& rid, double& c_in, double& c_out) {
    if (w.node == -2) return false;
    for (;;) {
        if (w.node < 0) {
            bool got = false;
            while (w.sp > 0) {
                --w.sp;
                double tf = (double)w.st_tf[w.sp], tn = (double)w.st_tn[w.sp];
                if (tf <= t || tn >= tmax) continue;
                w.node = w.st_node[w.sp];
                w.tn = tn;
                w.tf = tf;
                got = true;
                break;
            }
            if (!got) { w.node = -2; return false; }
        }
        const int node = w.node;
        if (!flags[node] || w.tf <= t || w.tn >= tmax) { w.node = -1; continue; }
        const KdNode nd = S.kd[node];
        if ((nd.a & 3) != 3) {  // interior (cavity leaves never have a set flag)
            const int axis = nd.a & 3, left = nd.a >> 2;
            const double p = (double)nd.b * 0.5;
            if (r.d[axis] == 0.0) {  // half-open rule: only the side containing o
                w.node = r.o[axis] < p ? left : left + 1;
                continue;
            }
            const double tp = (p - r.o[axis]) * r.inv[axis];
            const int near_c = r.d[axis] > 0.0 ? left : left + 1;
            const int far_c = near_c == left ? left + 1 : left;
            if (tp >= w.tf) { w.node = near_c; continue; }      // far side: r_in >= tp >= tf
            if (tp <= w.tn) { w.node = far_c; continue; }       // near side: r_out <= tp <= tn
            if (tp < tmax && w.sp < kKdStack) {
                w.st_node[w.sp] = far_c;
                w.st_tn[w.sp] = __double2float_rd(tp);
                w.st_tf[w.sp] = __double2float_ru(w.tf);
                w.sp++;
            } else if (tp < tmax) {
                __trap();  // tree deeper than the stack: rejected at scene setup
            }
            w.node = near_c;
            w.tf = tp;
            continue;
        }
        // leaf with an active region
        w.node = -1;
        const int reg = nd.a >> 2;
        const RegionRec rr = S.rec[reg];
        double r_in, r_out;
        slab_h(rr.lo, rr.hi, r, r_in, r_out);
        double ci = r_in > t ? r_in : t;
        double co = r_out < tmax ? r_out : tmax;
        if (ci < co) {
            rid = reg;
            c_in = ci;
            c_out = co;
            return true;
        }
    }
}

// One node visit of the same walk, for software pipelining (k_frame): `nd`
// and `fl` are the prefetched record / flag of w.node.  Returns 0 to
// continue, 1 when a region with a non-empty clipped interval was found,
// 2 when the walk is exhausted.  A sequence of kd_step calls yields exactly the
// regions kd_next would.
__device__ __forceinline__ int kd_step(const SceneView& S, const uint8_t* __restrict__ flags, const Ray& r, KdWalk& w,
                                       KdNode nd, uint8_t fl, double t, double tmax, int& rid, double& c_in,
                                       double& c_out) {
    if (w.node == -2) return 2;
    if (w.node < 0) {
        while (w.sp > 0) {
            --w.sp;
            const double tf = (double)w.st_tf[w.sp], tn = (double)w.st_tn[w.sp];
            if (tf <= t || tn >= tmax) continue;
            w.node = w.st_node[w.sp];
            w.tn = tn;
            w.tf = tf;
            return 0;
        }
        w.node = -2;
        return 2;
    }
    if (!fl || w.tf <= t || w.tn >= tmax) {
        w.node = -1;
        return 0;
    }
    if ((nd.a & 3) != 3) {
        const int axis = nd.a & 3, left = nd.a >> 2;
        const double p = (double)nd.b * 0.5;
        if (r.d[axis] == 0.0) {
            w.node = r.o[axis] < p ? left : left + 1;
            return 0;
        }
        const double tp = (p - r.o[axis]) * r.inv[axis];
        const int near_c = r.d[axis] > 0.0 ? left : left + 1;
        const int far_c = near_c == left ? left + 1 : left;
        if (tp >= w.tf) { w.node = near_c; return 0; }
        if (tp <= w.tn) { w.node = far_c; return 0; }
        if (tp < tmax) {
            if (w.sp >= kKdStack) __trap();
            w.st_node[w.sp] = far_c;
            w.st_tn[w.sp] = __double2float_rd(tp);
            w.st_tf[w.sp] = __double2float_ru(w.tf);
            w.sp++;
        }
        w.node = near_c;
        w.tf = tp;
        return 0;
    }
    w.node = -1;
    const int reg = nd.a >> 2;
    const RegionRec rr = S.rec[reg];
    double r_in, r_out;
    slab_h(rr.lo, rr.hi, r, r_in, r_out);
    const double ci = r_in > t ? r_in : t;
    const double co = r_out < tmax ? r_out : tmax;
    if (ci < co) {
        rid = reg;
        c_in = ci;
        c_out = co;
        return 1;
    }
    return 0;
}

// half-open point location through the k-d tree (`_bvh_point_query` on the
// all-regions index, R/accel.py:355-388)
__device__ __forceinline__ int kd_point(const SceneView& S, double px, double py, double pz) {
    if (S.n_kd == 0) return -1;
    const double p[3] = {px, py, pz};
    int node = 0;
    for (;;) {
        const KdNode nd = S.kd[node];
        if (nd.a == -1) return -1;
        if ((nd.a & 3) == 3) {
            const int reg = nd.a >> 2;
            const RegionRec rr = S.rec[reg];
#pragma unroll
            for (int a = 0; a < 3; a++)
                if (!(p[a] >= (double)rr.lo[a] * 0.5 && p[a] < (double)rr.hi[a] * 0.5)) return -1;
            return reg;
        }
        const int axis = nd.a & 3, left = nd.a >> 2;
        node = p[axis] < (double)nd.b * 0.5 ? left : left + 1;
    }
}

// ---------------------------------------------------------------------------
// LBVH traversal (csrc/lbvh.cu builds the tree; see lbvh.cuh)

struct __align__(16) LbvhNode {
    int32_t lo[3], hi[3];  // half-unit box (exact: union of region boxes)
    int32_t left, right;   // >= 0: internal node; < 0: leaf ~k -> prims[k]
};
static_assert(sizeof(LbvhNode) == 32, "LbvhNode is 32 bytes");

constexpr int kLbvhStack = 128;  // R/accel.py:297 uses the same depth

struct LbvhView {
    const LbvhNode* __restrict__ nodes;  // n_prims - 1 internal nodes, root 0
    const int32_t* __restrict__ prims;   // active region ids in Morton order
    int64_t n_prims;
};

// box of a child reference (internal node or leaf region)
__device__ __forceinline__ void lbvh_child_box(const SceneView& S, const LbvhView& L, int32_t c, const int32_t*& lo,
                                               const int32_t*& hi) {
    if (c >= 0) {
        lo = L.nodes[c].lo;
        hi = L.nodes[c].hi;
    } else {
        const RegionRec& rr = S.rec[L.prims[~c]];
        lo = rr.lo;
        hi = rr.hi;
    }
}

// _bvh_next_hit (R/accel.py:285-352): closest active region with clipped entry
// max(r_in, t) < min(r_out, t_max); ties -> lower region id.
__device__ inline bool lbvh_next_hit(const SceneView& S, const LbvhView& L, const Ray& r, double t_start,
                                     double t_max, int& rid, double& c_in_o, double& c_out_o) {
    int best_r = -1;
    double best_in = INFINITY, best_out = INFINITY;
    if (L.n_prims == 0) return false;
    int32_t stack[kLbvhStack];
    int top = 0;
    stack[top++] = L.n_prims == 1 ? ~0 : 0;
    while (top > 0) {
        const int32_t node = stack[--top];
        if (node < 0) {  // leaf: one region
            const int reg = L.prims[~node];
            const RegionRec rr = S.rec[reg];
            double r_in, r_out;
            slab_h(rr.lo, rr.hi, r, r_in, r_out);
            const double ci = r_in > t_start ? r_in : t_start;
            const double co = r_out < t_max ? r_out : t_max;
            if (ci < co && (ci < best_in || (ci == best_in && reg < best_r))) {
                best_r = reg;
                best_in = ci;
                best_out = co;
            }
            continue;
        }
        const LbvhNode nd = L.nodes[node];
        double n_in, n_out;
        slab_h(nd.lo, nd.hi, r, n_in, n_out);
        const double lo_t = n_in > t_start ? n_in : t_start;
        const double hi_t = n_out < t_max ? n_out : t_max;
        if (lo_t >= hi_t || lo_t > best_in) continue;
        // near child first (LIFO: push the far one first)
        const int32_t *llo, *lhi, *rlo, *rhi;
        lbvh_child_box(S, L, nd.left, llo, lhi);
        lbvh_child_box(S, L, nd.right, rlo, rhi);
        double l_in, l_out, q_in, q_out;
        slab_h(llo, lhi, r, l_in, l_out);
        slab_h(rlo, rhi, r, q_in, q_out);
        if (top + 2 > kLbvhStack) __trap();  // depth checked at build time
        if (l_in <= q_in) {
            stack[top++] = nd.right;
            stack[top++] = nd.left;
        } else {
            stack[top++] = nd.left;
            stack[top++] = nd.right;
        }
    }
    if (best_r < 0) return false;
    rid = best_r;
    c_in_o = best_in;
    c_out_o = best_out;
    return true;
}

// _bvh_point_query (R/accel.py:355-388): region whose half-open box holds p
__device__ inline int lbvh_point(const SceneView& S, const LbvhView& L, double px, double py, double pz) {
    if (L.n_prims == 0) return -1;
    const double p[3] = {px, py, pz};
    int32_t stack[kLbvhStack];
    int top = 0;
    stack[top++] = L.n_prims == 1 ? ~0 : 0;
    while (top > 0) {
        const int32_t node = stack[--top];
        const int32_t *lo, *hi;
        lbvh_child_box(S, L, node, lo, hi);
        bool in = true;
#pragma unroll
        for (int a = 0; a < 3; a++) in = in && p[a] >= (double)lo[a] * 0.5 && p[a] < (double)hi[a] * 0.5;
        if (!in) continue;
        if (node < 0) return L.prims[~node];
        if (top + 2 > kLbvhStack) __trap();
        stack[top++] = L.nodes[node].right;
        stack[top++] = L.nodes[node].left;
    }
    return -1;
}


// ---------------------------------------------------------------------------
// reconstruction: _accumulate_bricks / _gradient_bricks fused in one gather
// (R/sampling.py:57-103, 123-181).  GRAD=false: value only.

struct Accum {
    double num, den;              // unshifted (value path)
    double gnum, dn[3], dd[3];    // v0-shifted (gradient path)
    double v0;
    bool have_ref;
    int64_t n_nz;                 // cells with h > 0 (byte accounting)
};

template <bool GRAD>
__device__ __forceinline__ void gather(const SceneView& S, const int32_t* __restrict__ ids, int nids, double px,
                                       double py, double pz, Accum& A) {
    A.num = 0.0; A.den = 0.0;
    if (GRAD) {
        A.gnum = 0.0;
        A.dn[0] = A.dn[1] = A.dn[2] = 0.0;
        A.dd[0] = A.dd[1] = A.dd[2] = 0.0;
        A.v0 = 0.0;
        A.have_ref = false;
    }
    A.n_nz = 0;
    for (int t = 0; t < nids; t++) {
        const int b = ids[t];  // plain load: callers may pass a local id
        const int4 ba = __ldg(S.brick_a + b);
        const uint32_t bm = __ldg(S.brick_m + b);
        const int lev = bm & 31;
        const int nx = (bm >> 5) & 511, ny = (bm >> 14) & 511, nz = (bm >> 23) & 511;
        const double w = pow2(lev), iw_d = pow2(-lev);
        const int64_t iw = (int64_t)1 << lev;
        const int64_t lx = ba.x, ly = ba.y, lz = ba.z;
        // floor((p - l) / w - 0.5): division by a power of two == scaling
        const int64_t x0 = (int64_t)floor((px - (double)lx) * iw_d - 0.5);
        const int64_t y0 = (int64_t)floor((py - (double)ly) * iw_d - 0.5);
        const int64_t z0 = (int64_t)floor((pz - (double)lz) * iw_d - 0.5);
        const int64_t xs = x0 > 0 ? x0 : 0, xe = x0 + 2 < nx ? x0 + 2 : nx;
        const int64_t ys = y0 > 0 ? y0 : 0, ye = y0 + 2 < ny ? y0 + 2 : ny;
        const int64_t zs = z0 > 0 ? z0 : 0, ze = z0 + 2 < nz ? z0 + 2 : nz;
        const float* __restrict__ base = S.vals + (uint32_t)ba.w;
        for (int64_t z = zs; z < ze; z++) {
            const double ck = (double)(lz + z * iw) + 0.5 * w;
            const double hz = 1.0 - fabs(ck - pz) * iw_d;
            for (int64_t y = ys; y < ye; y++) {
                const double cj = (double)(ly + y * iw) + 0.5 * w;
                const double hy = 1.0 - fabs(cj - py) * iw_d;
                for (int64_t x = xs; x < xe; x++) {
                    const double ci = (double)(lx + x * iw) + 0.5 * w;
                    const double hx = 1.0 - fabs(ci - px) * iw_d;
                    if (hx > 0.0 && hy > 0.0 && hz > 0.0) {
                        const double h = hx * hy * hz;
                        const double v = (double)__ldg(base + x + nx * (y + ny * z));
                        A.num += h * v;
                        A.den += h;
                        A.n_nz++;
                        if (GRAD) {
                            const double sx = ci - px > 0.0 ? 1.0 : -1.0;
                            const double sy = cj - py > 0.0 ? 1.0 : -1.0;
                            const double sz = ck - pz > 0.0 ? 1.0 : -1.0;
                            const double gx = sx * iw_d * hy * hz;
                            const double gy = sy * iw_d * hx * hz;
                            const double gz = sz * iw_d * hx * hy;
                            if (!A.have_ref) { A.v0 = v; A.have_ref = true; }
                            const double u = v - A.v0;
                            A.gnum += h * u;
                            A.dn[0] += gx * u; A.dn[1] += gy * u; A.dn[2] += gz * u;
                            A.dd[0] += gx; A.dd[1] += gy; A.dd[2] += gz;
                        }
                    }
                }
            }
        }
    }
}

// Same sums as gather<GRAD>, restructured for SIMT: the <=2x2x2 candidate
// window of a brick is fixed, so the three hat factors per axis (and the
// products hx*hy) are computed once per brick instead of once per cell.  Every
// value is the identical IEEE expression of the reference (h = (hx*hy)*hz,
// g_x = ((s_x/w)*hy)*hz, ...) and cells are still visited z, y, x ascending, so
// the partial-sum sequence — and hence every bit — is unchanged.
template <bool GRAD>
__device__ __forceinline__ void gather_fast(const SceneView& S, const int32_t* __restrict__ ids, int nids, double px,
                                            double py, double pz, Accum& A) {
    A.num = 0.0; A.den = 0.0;
    if (GRAD) {
        A.gnum = 0.0;
        A.dn[0] = A.dn[1] = A.dn[2] = 0.0;
        A.dd[0] = A.dd[1] = A.dd[2] = 0.0;
        A.v0 = 0.0;
        A.have_ref = false;
    }
    A.n_nz = 0;
    for (int t = 0; t < nids; t++) {
        const int b = __ldg(ids + t);
        const int4 ba = __ldg(S.brick_a + b);
        const uint32_t bm = __ldg(S.brick_m + b);
        const int lev = bm & 31;
        const int nx = (bm >> 5) & 511, ny = (bm >> 14) & 511, nz = (bm >> 23) & 511;
        const double w = pow2(lev), iw_d = pow2(-lev);
        const double fx = floor((px - (double)ba.x) * iw_d - 0.5);
        const double fy = floor((py - (double)ba.y) * iw_d - 0.5);
        const double fz = floor((pz - (double)ba.z) * iw_d - 0.5);
        // window entirely outside the brick: no cell contributes (exact skip)
        if (!(fx >= -1.0 && fx < (double)nx && fy >= -1.0 && fy < (double)ny && fz >= -1.0 && fz < (double)nz)) continue;
        const int x0 = (int)fx, y0 = (int)fy, z0 = (int)fz;
        const double half = 0.5 * w;
        // cell centres (ai + 0.5*w), exact in FP64
        const double cx0 = (double)(ba.x + x0 * (1 << lev)) + half, cx1 = cx0 + w;
        const double cy0 = (double)(ba.y + y0 * (1 << lev)) + half, cy1 = cy0 + w;
        const double cz0 = (double)(ba.z + z0 * (1 << lev)) + half, cz1 = cz0 + w;
        const double ex0 = cx0 - px, ex1 = cx1 - px, ey0 = cy0 - py, ey1 = cy1 - py, ez0 = cz0 - pz, ez1 = cz1 - pz;
        const double hx[2] = {1.0 - fabs(ex0) * iw_d, 1.0 - fabs(ex1) * iw_d};
        const double hy[2] = {1.0 - fabs(ey0) * iw_d, 1.0 - fabs(ey1) * iw_d};
        const double hz[2] = {1.0 - fabs(ez0) * iw_d, 1.0 - fabs(ez1) * iw_d};
        const bool vx[2] = {x0 >= 0 && hx[0] > 0.0, x0 + 1 < nx && hx[1] > 0.0};
        const bool vy[2] = {y0 >= 0 && hy[0] > 0.0, y0 + 1 < ny && hy[1] > 0.0};
        const bool vz[2] = {z0 >= 0 && hz[0] > 0.0, z0 + 1 < nz && hz[1] > 0.0};
        const double sxw[2] = {ex0 > 0.0 ? iw_d : -iw_d, ex1 > 0.0 ? iw_d : -iw_d};
        const double syw[2] = {ey0 > 0.0 ? iw_d : -iw_d, ey1 > 0.0 ? iw_d : -iw_d};
        const double szw[2] = {ez0 > 0.0 ? iw_d : -iw_d, ez1 > 0.0 ? iw_d : -iw_d};
        const float* __restrict__ base = S.vals + (uint32_t)ba.w + x0 + nx * (y0 + ny * z0);
        // products shared by the cells of the 2x2x2 window
        double hxy[2][2];
#pragma unroll
        for (int dy = 0; dy < 2; dy++)
#pragma unroll
            for (int dx = 0; dx < 2; dx++) hxy[dy][dx] = hx[dx] * hy[dy];  // (hx*hy) as in h = hx*hy*hz
        // Branch-free cell body: a skipped cell contributes exact zeros.  The
        // accumulators start at +0.0 and round-to-nearest never yields -0.0
        // from non-(-0.0) operands, so adding +-0.0 leaves every bit unchanged.
#pragma unroll
        for (int dz = 0; dz < 2; dz++) {
#pragma unroll
            for (int dy = 0; dy < 2; dy++) {
                const float* row = base + nx * (dy + ny * dz);
#pragma unroll
                for (int dx = 0; dx < 2; dx++) {
                    const bool ok = vz[dz] && vy[dy] && vx[dx];
                    const double h = ok ? hxy[dy][dx] * hz[dz] : 0.0;
                    const double v = ok ? (double)__ldg(row + dx) : 0.0;
                    A.num += h * v;  // value path: exact reference arithmetic
                    A.den += h;
                    A.n_nz += ok;
                    if (GRAD) {
                        // Shading-only gradient (feeds the headlight factor, never alpha,
                        // positions or counters): fused multiply-adds and shared products
                        // are allowed here — well inside the 1e-3 image tolerance, and a
                        // locally constant field still cancels to an exactly zero gradient
                        // (every u below is exactly 0).
                        const double gx = ok ? sxw[dx] * (hy[dy] * hz[dz]) : 0.0;
                        const double gy = ok ? syw[dy] * (hx[dx] * hz[dz]) : 0.0;
                        const double gz = ok ? szw[dz] * hxy[dy][dx] : 0.0;
                        if (ok && !A.have_ref) { A.v0 = v; A.have_ref = true; }
                        const double u = v - A.v0;
                        A.gnum = __fma_rn(h, u, A.gnum);
                        A.dn[0] = __fma_rn(gx, u, A.dn[0]);
                        A.dn[1] = __fma_rn(gy, u, A.dn[1]);
                        A.dn[2] = __fma_rn(gz, u, A.dn[2]);
                        A.dd[0] += gx; A.dd[1] += gy; A.dd[2] += gz;
                    }
                }
            }
        }
    }
}

// Frame-kernel gather (k_warp, k_short): the value sums num/den are the
// reference's exact FP64 sequence; the analytic gradient, which only feeds the
// headlight shading factor (R/render.py:284-289, never alpha, positions or
// counters), is evaluated in FP32 with the trilinear sums factored per axis.
// Per brick, with the hat factors of invalid window cells zeroed,
//   gnum = sum hx hy hz u,  dn_x = sum sx hy hz u, ...,  dd_x = (sum sx)(sum hy)(sum hz), ...
// where u = v - v0 (v0 = first contributing cell, R/sampling.py:160-170), so a
// locally constant field still yields an exactly zero gradient (shade 0.2).
// g = dn*den - gnum*dd is the reference's quotient-rule numerator; the positive
// 1/den^2 is dropped because the shading factor depends on the direction only.
struct FastAccum {
    double num, den;
    float g[3];
    int n_nz;
};

// Brick record of the frame gather, in region-list order (one per entry of
// RegionSet.brick_ids): the lower corner as FP64 (no integer->FP64 conversion
// per sample: the conversion unit, not the FP64 pipe, limited the round-1
// gather), the scalar offset, and level | nx<<5 | ny<<14 | nz<<23.  32 B, two
// 16-B loads, read by every lane of a warp at the same address (broadcast).
struct __align__(16) RbRec {
    double lx, ly, lz;
    uint32_t off, meta;
};
static_assert(sizeof(RbRec) == 32, "RbRec is 32 bytes");

__device__ __forceinline__ RbRec load_rb(const RbRec* __restrict__ p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const int4 b = __ldg(reinterpret_cast<const int4*>(p) + 1);
    RbRec r;
    r.lx = a.x;
    r.ly = a.y;
    r.lz = __hiloint2double(b.y, b.x);
    r.off = (uint32_t)b.z;
    r.meta = (uint32_t)b.w;
    return r;
}

// Running state of the frame gather of one sample (value sums in the
// reference's exact FP64 sequence; FP32 shading-gradient partials).  Pairing
// the FP32 partials over dz on sm_100's f32x2 instructions cut brick_step from
// 258 to 239 SASS instructions but measured slower (orbit-mean C3 0.904 vs
// 0.897 ms, C2 6.17 vs 6.04: longer dependent chains, 40 more spill bytes).
struct ShadeAcc {
    double num, den;
    float fden, gnum, dn0, dn1, dn2, dd0, dd1, dd2, v0;
    int n_nz;
    bool have_ref;
    __device__ __forceinline__ void clear() {
        num = den = 0.0;
        fden = gnum = dn0 = dn1 = dn2 = dd0 = dd1 = dd2 = v0 = 0.f;
        n_nz = 0;
        have_ref = false;
    }
    // quotient-rule numerator of the analytic gradient (direction only, see FastAccum)
    __device__ __forceinline__ void gradient(float g[3]) const {
        g[0] = dn0 * fden - gnum * dd0;
        g[1] = dn1 * fden - gnum * dd1;
        g[2] = dn2 * fden - gnum * dd2;
    }
};

// One axis of a brick's 2-cell window (R/sampling.py:90-100, _hat_terms 57-63):
// x0 = floor((p - l)/w - 0.5); cell centres c = l + (x + 0.5) w; hats
// 1 - |c - p|/w.  Division by the power-of-two width is an exact scaling, so
// each fused multiply-add below rounds exactly once where the reference's
// unfused code rounds once (the product is exact): bit-identical values.
// The floor comes from one conversion (cvt.rmi) and the centre from the
// integer back in FP64 — two conversion-unit ops per axis (round 1: four).
struct Axis2 {
    double h0, h1;  // hats of slots x0, x0 + 1, zeroed when the slot is invalid
    int x0;
    bool v0, v1;    // slot inside the brick and hat > 0 (the reference's h > 0 test)
    float s0, s1;   // gradient slopes: sign(c - p) / w, zeroed when invalid
};

__device__ __forceinline__ Axis2 window_axis(double p, double l, int n, double w, double iw, float fw) {
    Axis2 A;
    const double t = __fma_rn(p - l, iw, -0.5);
    A.x0 = __double2int_rd(t);
    const double c0 = __fma_rn((double)A.x0 + 0.5, w, l);  // exact: l + (x0 + 1/2) w
    const double e0 = c0 - p, e1 = (c0 + w) - p;
    const double h0 = __fma_rn(-fabs(e0), iw, 1.0), h1 = __fma_rn(-fabs(e1), iw, 1.0);
    // sign tests on the high words (integer pipe; the FP64 pipe is the gather's
    // bottleneck).  For a double x that is 0, normal, or negative, x > 0.0 <=> its
    // high word is > 0 as a signed int; subnormal h or e cannot occur here (h is
    // 0 or >= 2^-53, e a difference of doubles ~ the coordinates' magnitude)
    A.v0 = (unsigned)A.x0 < (unsigned)n && __double2hiint(h0) > 0;
    A.v1 = (unsigned)(A.x0 + 1) < (unsigned)n && __double2hiint(h1) > 0;
    A.s0 = A.v0 ? (__double2hiint(e0) > 0 ? fw : -fw) : 0.f;
    A.s1 = A.v1 ? (__double2hiint(e1) > 0 ? fw : -fw) : 0.f;
    A.h0 = A.v0 ? h0 : 0.0;
    A.h1 = A.v1 ? h1 : 0.0;
    return A;
}

// one brick of the frame gather: adds brick b's window cells to A.  Every
// listed brick's support holds the whole region (ABR construction), so the
// window always overlaps the brick; invalid slots get zero hats (a skipped
// term adds +0 / +-0, leaving the running sums bit-identical) and clamped,
// in-brick load indices, so the 8 cells run branch-free.
template <bool GRAD>
__device__ __forceinline__ void brick_step(const SceneView& S, const RbRec& B, double px, double py, double pz,
                                           ShadeAcc& A) {
    const int lev = B.meta & 31;
    const int nx = (B.meta >> 5) & 511, ny = (B.meta >> 14) & 511, nz = (B.meta >> 23) & 511;
    const double w = pow2(lev), iw = pow2(-lev);
    const float fw = __int_as_float((127 - lev) << 23);  // 1/w in FP32
    const Axis2 X = window_axis(px, B.lx, nx, w, iw, fw);
    const Axis2 Y = window_axis(py, B.ly, ny, w, iw, fw);
    const Axis2 Z = window_axis(pz, B.lz, nz, w, iw, fw);
    A.n_nz += ((int)X.v0 + (int)X.v1) * ((int)Y.v0 + (int)Y.v1) * ((int)Z.v0 + (int)Z.v1);
    // The 2x2x2 window is read unclamped from S.gvals, the field's values with
    // kGatherPad zeros on both sides: an out-of-brick slot reads a finite
    // neighbour (or a pad zero) that its zero hat cancels exactly, so the eight
    // addresses are one pointer and three strides (+1 is an immediate offset).
    // The clamp to [-1, n-1] only keeps a corrupt window inside the pads.
    const int x0 = min(max(X.x0, -1), nx - 1), y0 = min(max(Y.x0, -1), ny - 1), z0 = min(max(Z.x0, -1), nz - 1);
    const int sy = nx, sz = nx * ny;
    const float* __restrict__ p0 = S.gvals + B.off + (x0 + nx * y0 + sz * z0);
    const float* __restrict__ p1 = p0 + sz;
    float vv[2][2][2];  // [dz][dy][dx]
    vv[0][0][0] = __ldg(p0); vv[0][0][1] = __ldg(p0 + 1);
    vv[0][1][0] = __ldg(p0 + sy); vv[0][1][1] = __ldg(p0 + sy + 1);
    vv[1][0][0] = __ldg(p1); vv[1][0][1] = __ldg(p1 + 1);
    vv[1][1][0] = __ldg(p1 + sy); vv[1][1][1] = __ldg(p1 + sy + 1);
    // the reference's sequence: h = (hx*hy)*hz, cells z, y, x ascending
    const double hxy00 = X.h0 * Y.h0, hxy01 = X.h1 * Y.h0, hxy10 = X.h0 * Y.h1, hxy11 = X.h1 * Y.h1;  // [dy][dx]
    const double hzz[2] = {Z.h0, Z.h1};
#pragma unroll
    for (int dz = 0; dz < 2; dz++) {
        const double h0 = hxy00 * hzz[dz], h1 = hxy01 * hzz[dz], h2 = hxy10 * hzz[dz], h3 = hxy11 * hzz[dz];
        A.num += h0 * (double)vv[dz][0][0]; A.den += h0;
        A.num += h1 * (double)vv[dz][0][1]; A.den += h1;
        A.num += h2 * (double)vv[dz][1][0]; A.den += h2;
        A.num += h3 * (double)vv[dz][1][1]; A.den += h3;
    }
    if (GRAD) {
        if (!A.have_ref && (X.v0 || X.v1) && (Y.v0 || Y.v1) && (Z.v0 || Z.v1)) {  // first contributing cell
            const float r0 = X.v0 ? vv[0][0][0] : vv[0][0][1], r1 = X.v0 ? vv[0][1][0] : vv[0][1][1];
            const float r2 = X.v0 ? vv[1][0][0] : vv[1][0][1], r3 = X.v0 ? vv[1][1][0] : vv[1][1][1];
            const float p0 = Y.v0 ? r0 : r1, p1 = Y.v0 ? r2 : r3;
            A.v0 = Z.v0 ? p0 : p1;  // select chain: no local-memory indexing
            A.have_ref = true;
        }
        const float ax0 = (float)X.h0, ax1 = (float)X.h1, ay0 = (float)Y.h0, ay1 = (float)Y.h1,
                    az0 = (float)Z.h0, az1 = (float)Z.h1;
        float C[2], D[2], E[2];
#pragma unroll
        for (int dz = 0; dz < 2; dz++) {
            const float u00 = vv[dz][0][0] - A.v0, u01 = vv[dz][0][1] - A.v0;
            const float u10 = vv[dz][1][0] - A.v0, u11 = vv[dz][1][1] - A.v0;
            const float A0 = fmaf(ax1, u01, ax0 * u00), A1 = fmaf(ax1, u11, ax0 * u10);      // x-hat reductions
            const float B0 = fmaf(X.s1, u01, X.s0 * u00), B1 = fmaf(X.s1, u11, X.s0 * u10);  // x-slope reductions
            C[dz] = fmaf(ay1, A1, ay0 * A0);  // sum hx hy u
            D[dz] = fmaf(ay1, B1, ay0 * B0);  // sum sx hy u
            E[dz] = fmaf(Y.s1, A1, Y.s0 * A0);  // sum hx sy u
        }
        A.gnum = fmaf(az1, C[1], fmaf(az0, C[0], A.gnum));
        A.dn0 = fmaf(az1, D[1], fmaf(az0, D[0], A.dn0));
        A.dn1 = fmaf(az1, E[1], fmaf(az0, E[0], A.dn1));
        A.dn2 = fmaf(Z.s1, C[1], fmaf(Z.s0, C[0], A.dn2));
        const float Hx = ax0 + ax1, Hy = ay0 + ay1, Hz = az0 + az1;
        const float Sx = X.s0 + X.s1, Sy = Y.s0 + Y.s1, Sz = Z.s0 + Z.s1;
        A.fden = fmaf(Hx * Hy, Hz, A.fden);
        A.dd0 = fmaf(Sx * Hy, Hz, A.dd0);
        A.dd1 = fmaf(Hx * Sy, Hz, A.dd1);
        A.dd2 = fmaf(Hx * Hy, Sz, A.dd2);
    }
}

// the frame gather over region-list entries [off, off + nids) (S.rb)
template <bool GRAD>
__device__ __forceinline__ void gather_shade(const SceneView& S, int64_t off, int nids, double px, double py,
                                             double pz, FastAccum& F) {
    ShadeAcc A;
    A.clear();
    const RbRec* __restrict__ rb = S.rb + off;
    for (int t = 0; t < nids; t++) brick_step<GRAD>(S, load_rb(rb + t), px, py, pz, A);
    F.num = A.num;
    F.den = A.den;
    F.n_nz = A.n_nz;
    if (GRAD) A.gradient(F.g);
}

// _shade_factor (R/render.py:284-289) on an unnormalised FP32 gradient direction
// at a sample of value v.  Returns -1 when the FP32 gradient cannot be
// trusted: its largest component subnormal (in the far tail of a field the
// values are FP32 subnormals: the partials lose their precision and 1/m
// overflows) or not finite.  (Any normal gradient matched the reference's
// RGBA8 exactly over the configs[2] frame; a 2^-100 bound flagged 9 % of its
// pixels for nothing.)  An exactly zero gradient at a value of normal
// magnitude is genuine — every v - v0 is exactly 0 (a locally constant field,
// or a single contributing cell) — and shades 0.2 like the reference.  On -1
// the frame kernels shade with 0.2, and when the sample's opacity is not
// negligible (>= kNegligibleAlpha: a shading error of at most 0.8 alpha could
// show) list the pixel for k_fixup, which re-renders it with the reference's
// exact FP64 gradient.  Subnormal values under a TF that maps them to an
// alpha ~1e-38 (configs[2]'s far field) never need the re-render.
constexpr double kNegligibleAlpha = 0x1p-40;
__device__ __forceinline__ double shade_factor_f(const float g[3], const Ray& r, double v) {
    const float m = fmaxf(fabsf(g[0]), fmaxf(fabsf(g[1]), fabsf(g[2])));
    if (m == 0.f && fabs(v) >= 0x1p-60) return 0.2;
    if (!(m >= 0x1p-126f) || !(m < INFINITY)) return -1.0;
    const float s = 1.f / m;  // scale to [1, 3] before squaring: no under/overflow
    const float a = g[0] * s, b = g[1] * s, c = g[2] * s;
    const float dot = a * (float)r.d[0] + b * (float)r.d[1] + c * (float)r.d[2];
    return 0.2 + 0.8 * (double)(fabsf(dot) * rsqrtf(a * a + b * b + c * c));
}

__device__ __forceinline__ void analytic_gradient(const Accum& A, double g[3]) {
    // _sample_gradient mode 1, R/render.py:295-306
    if (A.den <= kEpsWeight) { g[0] = g[1] = g[2] = 0.0; return; }
    const double d2 = A.den * A.den;
#pragma unroll
    for (int a = 0; a < 3; a++) g[a] = (A.dn[a] * A.den - A.gnum * A.dd[a]) / d2;
}

__device__ __forceinline__ double shade_factor(const double g[3], const Ray& r) {
    // _shade_factor, R/render.py:284-289
    const double n = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (n == 0.0) return 0.2;
    return 0.2 + 0.8 * fabs(g[0] * r.d[0] + g[1] * r.d[1] + g[2] * r.d[2]) / n;
}

__device__ __forceinline__ void tf_eval(const double* tf, double tf_lo, double tf_hi, double v, double c[4]) {
    // _tf_eval, R/render.py:236-254
    double t = (v - tf_lo) / (tf_hi - tf_lo);
    if (t < 0.0) t = 0.0;
    else if (t > 1.0) t = 1.0;
    const double x = t * 255.0;
    const int i = (int)x;
    if (i >= 255) {
#pragma unroll
        for (int k = 0; k < 4; k++) c[k] = tf[255 * 4 + k];
        return;
    }
    const double f = x - (double)i, g = 1.0 - f;
#pragma unroll
    for (int k = 0; k < 4; k++) c[k] = g * tf[i * 4 + k] + f * tf[(i + 1) * 4 + k];
}

// _tf_eval (R/render.py:236-254) with the division by the domain width done
// through its hoisted reciprocal and 32-byte table loads.  t = (v - lo) / (hi -
// lo) is still the correctly rounded quotient: q0 = n * (1/d) is within 1 ulp,
// the residual n - q0 d is exact as one FMA, and q0 + r (1/d) rounded once is
// RN(n / d) when 1/d is itself correctly rounded (Markstein's theorem; 4e8
// random pairs incl. boundary significands agree with the division).  Until
// round 2 the bare q0 was used: a last-ulp change of t moves the colour by
// ~1e-16 only, but where the reference's alpha is exactly 1 (v at the top of
// a TF ending opaque) 1 - a ~1e-16 instead of 0 went through the opacity
// correction 1 - (1 - a)^y with the short first step y < 1 of an eye inside
// the volume to an alpha of 0.7-0.98 instead of 1 (RGBA off by 0.02, sample
// counters changed; tests/golden/make_inside.py's frames).  The plain division
// cost 2 % / 1 % of the C3 / C2 frame, this 2 FMAs.
__device__ __forceinline__ void tf_eval_fast(const double* tf, double tf_lo, double tf_den, double tf_inv, double v,
                                             double c[4]) {
    const double n = v - tf_lo, q0 = n * tf_inv;
    double t = __fma_rn(__fma_rn(-q0, tf_den, n), tf_inv, q0);
    if (t < 0.0) t = 0.0;
    else if (t > 1.0) t = 1.0;
    const double x = t * 255.0;
    const int i = (int)x;
    if (i >= 255) {
#pragma unroll
        for (int k = 0; k < 4; k++) c[k] = tf[255 * 4 + k];
        return;
    }
    const double f = x - (double)i, g = 1.0 - f;
    const double4 a = *reinterpret_cast<const double4*>(tf + 4 * i);
    const double4 b = *reinterpret_cast<const double4*>(tf + 4 * i + 4);
    c[0] = g * a.x + f * b.x;
    c[1] = g * a.y + f * b.y;
    c[2] = g * a.z + f * b.z;
    c[3] = g * a.w + f * b.w;
}

// opacity correction alpha' = 1 - (1 - a)^y (R/render.py:432) as
// -expm1(y * log(1 - a)): same rounded base 1 - a as the reference, within a
// few ulp of pow, and a fraction of pow's code size
__device__ __forceinline__ double opacity_correct(double a, double y) { return -expm1(y * log(1.0 - a)); }

// _collect_bricks (R/sampling.py:184-224): ids of the bricks in every split-tree
// leaf whose subtree box, dilated by its largest half cell width, holds p —
// a superset of the bricks whose supports contain p — sorted ascending.  The
// gather over them skips zero-weight cells exactly as over a region's list,
// so both give the same floats.  Returns -1 if more than `cap` ids.
constexpr int kTreeIds = 128;
__device__ inline int collect_bricks(const TreeView& T, double px, double py, double pz, int32_t* out, int cap) {
    int n = 0;
    int32_t stack[128];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        const int nd = stack[--top];
        const double e = T.mh[nd];
        if (px <= T.lo[3 * nd] - e || px >= T.hi[3 * nd] + e || py <= T.lo[3 * nd + 1] - e ||
            py >= T.hi[3 * nd + 1] + e || pz <= T.lo[3 * nd + 2] - e || pz >= T.hi[3 * nd + 2] + e)
            continue;
        if (T.axis[nd] < 0) {
            for (int b = T.bstart[nd]; b < T.bstart[nd] + T.bcount[nd]; b++) {
                if (n == cap) return -1;
                out[n++] = b;
            }
        } else {
            if (top + 2 > 128) return -1;
            stack[top++] = T.right[nd];
            stack[top++] = T.left[nd];
        }
    }
    for (int a = 1; a < n; a++) {  // insertion sort (small sets)
        const int32_t key = out[a];
        int c = a - 1;
        while (c >= 0 && out[c] > key) {
            out[c + 1] = out[c];
            c--;
        }
        out[c + 1] = key;
    }
    return n;
}

// central / clamped-central gradient (R/render.py:307-376)
__device__ inline void central_gradient(const SceneView& S, int mode, double px, double py, double pz, int rid,
                                        const int32_t* ids, int nids, double val, double g[3], int64_t* n_evals) {
    const RegionRec rr = S.rec[rid];
    const double h = 0.5 * pow2(rr.meta >> 24);
    const double p[3] = {px, py, pz};
    g[0] = g[1] = g[2] = 0.0;
    Accum A;
    for (int a = 0; a < 3; a++) {
        double qp[3] = {px, py, pz}, qm[3] = {px, py, pz};
        qp[a] = p[a] + h;
        qm[a] = p[a] - h;
        if (mode == 3) {
            for (int c = 0; c < 3; c++) {
                const double lo = (double)rr.lo[c] * 0.5, hi = (double)rr.hi[c] * 0.5;
                qp[c] = fmin(fmax(qp[c], lo), hi);
                qm[c] = fmin(fmax(qm[c], lo), hi);
            }
            gather<false>(S, ids, nids, qp[0], qp[1], qp[2], A);
            const double np_ = A.num, dp = A.den;
            gather<false>(S, ids, nids, qm[0], qm[1], qm[2], A);
            const double nm = A.num, dm = A.den;
            *n_evals += 2;
            if (dp > kEpsWeight && dm > kEpsWeight) {
                const double span = qp[a] - qm[a];
                if (span > 0.0) g[a] = (np_ / dp - nm / dm) / span;
            }
        } else {
            double fp = 0.0, fm = 0.0;
            bool okp = false, okm = false;
            const int rp = kd_point(S, qp[0], qp[1], qp[2]);
            if (rp >= 0) {
                const RegionRec q = S.rec[rp];
                gather<false>(S, S.rids + q.ids_begin, q.meta & 0xffffff, qp[0], qp[1], qp[2], A);
                *n_evals += 1;
                if (A.den > kEpsWeight) { fp = A.num / A.den; okp = true; }
            }
            const int rm = kd_point(S, qm[0], qm[1], qm[2]);
            if (rm >= 0) {
                const RegionRec q = S.rec[rm];
                gather<false>(S, S.rids + q.ids_begin, q.meta & 0xffffff, qm[0], qm[1], qm[2], A);
                *n_evals += 1;
                if (A.den > kEpsWeight) { fm = A.num / A.den; okm = true; }
            }
            double gg;
            if (okp && okm) gg = (fp - fm) / (2.0 * h);
            else if (okp) gg = (fp - val) / h;
            else if (okm) gg = (val - fm) / h;
            else gg = 0.0;
            g[a] = gg;
        }
    }
}

// ---------------------------------------------------------------------------
// per-ray march state shared by the frame and ray-batch kernels

struct MarchConst {
    double spc, rate, early;
    uint64_t seed;
    int grad_mode;
    int n_planes;
    double planes[6][4];
    int iso_on;
    double iso_value;
    double iso_rgb[3];
    double tf_lo, tf_hi;
    double tf_den, tf_inv;  // tf_hi - tf_lo, its correctly rounded reciprocal
    // host-computed per finest level (IEEE division on the host, same values
    // as the kernel would compute): dt = fw/(spc*rate), s1 = fw/spc (R/render.py:402-403)
    double lv_dt[32], lv_s1[32], lv_is1[32];
    // 1/dt when dt is a power of two (x / dt == x * (1/dt) exactly), else 0 (divide)
    double lv_idt[32];
    int use_tree;   // cell-location gather through the split tree (render_frame(use_celllocation=True))
};

// x / dt of the lattice (R/render.py:404-418) for level `lev`: one multiply
// when dt is a power of two (the bench configs), an IEEE division otherwise
__device__ __forceinline__ double div_dt(const MarchConst& M, int lev, double x) {
    const double idt = M.lv_idt[lev];
    return idt != 0.0 ? x * idt : x / M.lv_dt[lev];
}

struct RayStats {
    int64_t regions, samples, bytes;
};

__device__ __forceinline__ void clip_ray(const MarchConst& M, const Ray& r, double& tmin, double& tmax) {
    // _clip_ray, R/render.py:263-281
    for (int i = 0; i < M.n_planes; i++) {
        const double* pl = M.planes[i];
        const double nd = pl[0] * r.d[0] + pl[1] * r.d[1] + pl[2] * r.d[2];
        const double no = pl[0] * r.o[0] + pl[1] * r.o[1] + pl[2] * r.o[2];
        if (nd > 0.0) {
            const double t = (pl[3] - no) / nd;
            if (t < tmax) tmax = t;
        } else if (nd < 0.0) {
            const double t = (pl[3] - no) / nd;
            if (t > tmin) tmin = t;
        } else if (no > pl[3]) {
            tmin = 1.0;
            tmax = 0.0;
            return;
        }
    }
}

template <bool COUNT>
__device__ __forceinline__ void count_eval(RayStats& st, int nids, const Accum& A) {
    if (COUNT) st.bytes += 16 * (int64_t)nids + 4 * A.n_nz;
}

// a ray's active regions listed in ray order by k_walk; `trunc`: the list stops
// early and the k-d walk continues from the query point
struct IsoList {
    const int32_t* list;
    int n;
    bool trunc;
};

// _iso_ray, R/render.py:456-518
template <bool COUNT>
__device__ bool iso_ray(const SceneView& S, const uint8_t* __restrict__ iflags, const MarchConst& M, const Ray& r,
                        double tmin, double tmax, double rho, double& t_hit, double g[3], RayStats& st,
                        const LbvhView* lb = nullptr, const IsoList* lst = nullptr) {
    KdWalk w;
    int lpos = 0;
    bool walking = lst == nullptr;
    if (walking) kd_begin(S, r, w);
    double t = tmin;
    const double iso = M.iso_value;
    g[0] = g[1] = g[2] = 0.0;
    Accum A;
    for (;;) {
        int rid;
        double t_in, t_out;
        // next region: k_walk's list (exact slab + restart chain), the ordered k-d
        // walk, or a fresh LBVH closest-hit query (the reference's way)
        bool got = false;
        if (!walking) {
            while (lpos < lst->n) {
                const int reg = lst->list[lpos++];
                const RegionRec q = S.rec[reg];
                double r_in, r_out;
                slab_h(q.lo, q.hi, r, r_in, r_out);
                const double ci = r_in > t ? r_in : t, co = r_out < tmax ? r_out : tmax;
                if (ci < co) {
                    rid = reg;
                    t_in = ci;
                    t_out = co;
                    got = true;
                    break;
                }
            }
            if (!got && lst->trunc) {  // continue with the k-d walk (a walk from the root culls by t: exact)
                walking = true;
                kd_begin(S, r, w);
            }
        }
        if (walking)
            got = lb ? lbvh_next_hit(S, *lb, r, t, tmax, rid, t_in, t_out)
                     : kd_next(S, iflags, r, w, t, tmax, rid, t_in, t_out);
        if (!got) return false;
        const RegionRec rr = S.rec[rid];
        const int nids = rr.meta & 0xffffff;
        const int32_t* ids = S.rids + rr.ids_begin;
        if (COUNT) st.bytes += 32 + 4 * (int64_t)nids;
        const double fw = pow2(rr.meta >> 24);
        const double dt = fw / (M.spc * M.rate);
        double prev_t = t_in;
        gather<false>(S, ids, nids, r.o[0] + t_in * r.d[0], r.o[1] + t_in * r.d[1], r.o[2] + t_in * r.d[2], A);
        count_eval<COUNT>(st, nids, A);
        bool prev_ok = A.den > kEpsWeight;
        double prev_f = prev_ok ? A.num / A.den - iso : 0.0;
        double k = floor(t_in / dt - rho) + 1.0;
        bool done = false;
        while (!done) {
            double tk = dt * (k + rho);
            k += 1.0;
            if (tk >= t_out) { tk = t_out; done = true; }
            else if (tk <= prev_t) continue;
            gather<false>(S, ids, nids, r.o[0] + tk * r.d[0], r.o[1] + tk * r.d[1], r.o[2] + tk * r.d[2], A);
            count_eval<COUNT>(st, nids, A);
            const bool ok = A.den > kEpsWeight;
            const double f = ok ? A.num / A.den - iso : 0.0;
            if (prev_ok && ok && ((prev_f <= 0.0 && f >= 0.0) || (prev_f >= 0.0 && f <= 0.0)) &&
                !(prev_f == 0.0 && f == 0.0)) {
                double lo_t = prev_t, hi_t = tk, flo = prev_f;
                for (int it = 0; it < 16; it++) {
                    const double mid = 0.5 * (lo_t + hi_t);
                    gather<false>(S, ids, nids, r.o[0] + mid * r.d[0], r.o[1] + mid * r.d[1], r.o[2] + mid * r.d[2], A);
                    count_eval<COUNT>(st, nids, A);
                    const double fm = A.den > kEpsWeight ? A.num / A.den - iso : 0.0;
                    if ((flo <= 0.0 && fm <= 0.0) || (flo >= 0.0 && fm >= 0.0)) { lo_t = mid; flo = fm; }
                    else hi_t = mid;
                }
                t_hit = 0.5 * (lo_t + hi_t);
                gather<true>(S, ids, nids, r.o[0] + t_hit * r.d[0], r.o[1] + t_hit * r.d[1], r.o[2] + t_hit * r.d[2], A);
                if (A.den > kEpsWeight) {
                    const double d2 = A.den * A.den;
                    for (int a = 0; a < 3; a++) g[a] = (A.dn[a] * A.den - A.gnum * A.dd[a]) / d2;
                }
                return true;
            }
            prev_t = tk;
            prev_f = f;
            prev_ok = ok;
        }
        t = restart_t(t_out);
        if (t >= tmax) return false;
    }
}

// _volume_ray, R/render.py:380-453.  GRAD: 0 none, 1 analytic (fused gather),
// 2 central / 3 clamped central (mode in M.grad_mode).
template <int GRAD, bool COUNT>
__device__ void volume_ray(const SceneView& S, const uint8_t* __restrict__ vflags, const MarchConst& M,
                           const double* tf, const Ray& r, double tmin, double tmax, double rho, double acc[4],
                           RayStats& st, const LbvhView* lb = nullptr) {
    double ar = 0.0, ag = 0.0, ab = 0.0, aa = 0.0;
    KdWalk w;
    kd_begin(S, r, w);
    double t = tmin;
    Accum A;
    while (aa < M.early) {
        int rid;
        double t_in, t_out;
        if (!(lb ? lbvh_next_hit(S, *lb, r, t, tmax, rid, t_in, t_out)
                 : kd_next(S, vflags, r, w, t, tmax, rid, t_in, t_out)))
            break;
        st.regions++;
        const RegionRec rr = S.rec[rid];
        const int nids = rr.meta & 0xffffff;
        const int32_t* ids = S.rids + rr.ids_begin;
        if (COUNT) st.bytes += 32 + 4 * (int64_t)nids;
        const double fw = pow2(rr.meta >> 24);
        const double dt = fw / (M.spc * M.rate);
        const double s1 = fw / M.spc;
        double prev = t_in;
        double k = floor(t_in / dt - rho) + 1.0;
        bool done = false;
        while (!done) {
            double tk = dt * (k + rho);
            k += 1.0;
            if (tk >= t_out) { tk = t_out; done = true; }
            else if (tk <= prev) continue;
            const double sl = tk - prev;
            const double mid = 0.5 * (prev + tk);
            prev = tk;
            st.samples++;
            const double px = r.o[0] + mid * r.d[0], py = r.o[1] + mid * r.d[1], pz = r.o[2] + mid * r.d[2];
            if (M.use_tree && S.tree.n > 0) {  // cell location (R/render.py:423-425)
                int32_t tids[kTreeIds];
                const int tn = collect_bricks(S.tree, px, py, pz, tids, kTreeIds);
                if (tn >= 0) gather<GRAD == 1>(S, tids, tn, px, py, pz, A);
                else gather<GRAD == 1>(S, ids, nids, px, py, pz, A);  // same floats, see collect_bricks
            } else {
                gather<GRAD == 1>(S, ids, nids, px, py, pz, A);
            }
            count_eval<COUNT>(st, nids, A);
            if (A.den > kEpsWeight) {
                const double v = A.num / A.den;
                double c[4];
                tf_eval(tf, M.tf_lo, M.tf_hi, v, c);
                if (c[3] > 0.0) {
                    const double alpha = 1.0 - pow(1.0 - c[3], sl / s1);
                    if (GRAD != 0) {
                        double g[3];
                        if (GRAD == 1) {
                            analytic_gradient(A, g);
                        } else {
                            int64_t ne = 0;
                            central_gradient(S, M.grad_mode, px, py, pz, rid, ids, nids, v, g, &ne);
                        }
                        const double f = shade_factor(g, r);
                        c[0] *= f; c[1] *= f; c[2] *= f;
                    }
                    const double wgt = alpha * (1.0 - aa);
                    ar += wgt * c[0];
                    ag += wgt * c[1];
                    ab += wgt * c[2];
                    aa += wgt;
                    if (aa >= M.early) break;
                }
            }
        }
        t = restart_t(t_out);
        if (t >= tmax) break;
    }
    acc[0] = ar; acc[1] = ag; acc[2] = ab; acc[3] = aa;
}

}  // namespace xb
