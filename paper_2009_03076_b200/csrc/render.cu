// render.cu — the fused sm_100a ray-march kernels (paper §4-5) and the
// single-ray batch kernel behind integrate_ray / iso_intersect.
//
// Frame pipeline: k_classify -> CUB hit select -> k_walk ->
// k_route -> k_walk2 -> k_warp (warp per long ray, then a lane per short
// ray); iso scenes run the same chain on the iso set first, ending in
// k_iso_warp.  k_render: one thread per pixel, one block per tile — the
// kernel of the per-visit LBVH traversal and the cell-location gather
// (tuning.kernel = 1 runs every frame through it).
//
// The per-pixel arithmetic is `_render_kernel` (R/render.py:521-578) in both.
#include <cmath>
#include <memory>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>

#include "march.cuh"

#include "render.cuh"

namespace xb {

// ---------------------------------------------------------------------------
// slot -> pixel mapping (shared by both kernels and k_iso_pass)

struct SlotPix {
    int x, y;
    int64_t pix, out;
    bool live;
};

__device__ __forceinline__ SlotPix slot_pixel(const RenderArgs& A, int64_t slot) {
    SlotPix s;
    const int64_t t_local = slot / (kTileW * kTileH);
    const int local = (int)(slot % (kTileW * kTileH));
    const int wsub = local >> 5, ln = local & 31;
    const int lx = (wsub & 1) * 8 + (ln & 7);
    const int ly = (wsub >> 1) * 4 + (ln >> 3);
    const int64_t tile = (int64_t)A.tile_rank + t_local * A.tile_world;
    const int tx = (int)(tile % A.tiles_x), ty = (int)(tile / A.tiles_x);
    s.x = tx * kTileW + lx;
    s.y = ty * kTileH + ly;
    s.live = tile < (int64_t)A.tiles_x * A.tiles_y && s.x < A.W && s.y < A.H;
    s.pix = (int64_t)s.y * A.W + s.x;
    s.out = A.packed ? t_local * (kTileW * kTileH) + ly * kTileW + lx : s.pix;
    return s;
}

__device__ __forceinline__ void pixel_ray(const RenderArgs& A, int x, int y, Ray& r) {
    const double sx = (2.0 * ((double)x + 0.5) / (double)A.W - 1.0) * A.tan_half * A.aspect;
    const double sy = (1.0 - 2.0 * ((double)y + 0.5) / (double)A.H) * A.tan_half;
#pragma unroll
    for (int a = 0; a < 3; a++) r.d[a] = A.fwd[a] + sx * A.right[a] + sy * A.up[a];
    const double inv = 1.0 / sqrt(r.d[0] * r.d[0] + r.d[1] * r.d[1] + r.d[2] * r.d[2]);
#pragma unroll
    for (int a = 0; a < 3; a++) {
        r.d[a] *= inv;
        r.o[a] = A.pos[a];
        r.inv[a] = 1.0 / r.d[a];
    }
}

__device__ __forceinline__ void write_pixel(const RenderArgs& A, int64_t out, const double acc[4], int nreg,
                                            int nsmp) {
    uchar4 q;
    unsigned char* qc = reinterpret_cast<unsigned char*>(&q);
#pragma unroll
    for (int c = 0; c < 4; c++) {
        double v = acc[c] < 0.0 ? 0.0 : acc[c];
        v = v > 1.0 ? 1.0 : v;
        qc[c] = (unsigned char)(v * 255.0 + 0.5);
    }
    A.out8[out] = q;
    if (A.outf) A.outf[out] = make_double4(acc[0], acc[1], acc[2], acc[3]);
    if (A.outcnt) A.outcnt[out] = make_int2(nreg, nsmp);
}

// ---------------------------------------------------------------------------
// iso pre-pass: t_hit and headlight factor per slot (the iso ray runs first
// and bounds the volume ray, R/render.py:551-558)

template <bool COUNT>
__global__ void __launch_bounds__(128) k_iso_pass(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= n_slots) return;
    const SlotPix sp = slot_pixel(A, slot);
    double t_end = -1.0, f = -1.0;
    RayStats st = {0, 0, 0};
    if (sp.live) {
        Ray r;
        pixel_ray(A, sp.x, sp.y, r);
        const double rho = rho_hash((uint64_t)sp.pix, A.M.seed);
        double tmin = 0.0, tmax = kTFar;
        clip_ray(A.M, r, tmin, tmax);
        t_end = tmax;
        if (tmin < tmax) {
            double g[3], th = 0.0;
            if (iso_ray<COUNT>(A.S, A.iflags, A.M, r, tmin, tmax, rho, th, g, st, A.use_lbvh ? &A.ilb : nullptr)) {
                t_end = th;
                f = shade_factor(g, r);
            }
        }
    }
    A.iso_tend[slot] = t_end;
    A.iso_shade[slot] = f;
    if (COUNT && st.bytes) atomicAdd(&A.stats[2], (unsigned long long)st.bytes);
}

// ---------------------------------------------------------------------------
// k_warp: one warp per ray (default kernel).
//
// Traversal is a warp-cooperative *ordered frontier* over the region k-d tree:
// lane i holds the i-th entry of an ordered list of disjoint subtrees that
// together cover the rest of the ray (front-to-back order).  One expansion
// step loads the node of every unresolved entry at once (32 independent loads
// instead of one dependent chain) and replaces it in place by its children
// (near child first) or drops it (culled / inactive); resolved leaves keep
// their place.  The list tail beyond 32 entries spills to a per-warp LIFO in
// shared memory — every spilled entry lies after everything in the frontier
// and before everything spilled earlier, so popping restores list order.
// Culling is the same conservative test as kd_next, so the leaves come out in
// exactly r_in order.
//
// The leading run of leaves is then consumed as a batch: exact slab test per
// lane, the reference's restart chain t_i = restart(t_out of the previous
// visited region) (R/render.py:451-453), the lattice count of every segment,
// a warp prefix sum, and the samples in chunks of 32 — every lane takes one
// sample of the ray, so the gather runs converged.  Compositing a chunk is a
// warp scan of the front-to-back "over" operator (T, C) -> (T_a T_b, C_a +
// T_a C_b); the first lane whose accumulated alpha reaches `early` ends the
// ray, and the sample / region counters stop exactly there (R/render.py:419,
// 448-449).  The scan reassociates the alpha recurrence, so alpha differs from
// the reference by rounding only (~1e-16), like CUDA's pow.

#ifndef XB_WARP_THREADS
#define XB_WARP_THREADS 128
#endif
constexpr int kWarpThreads = XB_WARP_THREADS;
#ifndef XB_WARP_MINB
#define XB_WARP_MINB 4
#endif
constexpr int kWarpMinBlocks = XB_WARP_MINB;
constexpr int kWarpsPerBlock = kWarpThreads / 32;
constexpr int kWarpStack = 256;  // spilled frontier entries per warp
constexpr int kRaysPerGrab = 8;  // rays taken per work-counter atomic
// A (sample, brick)-flattened chunk gather (each lane one brick per round,
// partials combined through shared memory) measured slower every time — C2
// 12.3 vs 10.1 ms (first pipeline), C3 1.21 vs 0.92 and C2 8.74 vs 6.31 (walk
// lists): the per-round barriers and the combine loop cost more than the idle
// lane-brick slots of the per-sample loop.  Removed in round 2.  Round 2 also
// measured "helper lanes" — a partial chunk's idle lane m + j gathering the
// later half of sample j's brick list, merged by shuffles (one convergent
// loop): orbit-mean C3 0.927 vs 0.897 ms, C2 6.40 vs 6.04 — slower as well
// (the merge state and shuffles cost more than the idle lanes).

struct SegQ {       // one visited region of the segment queue
    double ci, co;   // clipped interval
    double kf;       // first lattice index inside (t_in, t_out)
    int ids, meta;   // RegionRec.ids_begin / meta
    int cnt, rid;    // samples, region id
};

struct SpillEnt {
    int code;        // >= 0: unresolved k-d node; <= -2: resolved leaf, region -2 - code
    float tn, tf;    // conservative ray interval of the subtree (rounded outward)
};

__device__ __forceinline__ double sel3(int a, const double v[3]) { return a == 0 ? v[0] : (a == 1 ? v[1] : v[2]); }
__device__ __forceinline__ double sel4(int i, const double v[4]) {
    return i < 2 ? (i == 0 ? v[0] : v[1]) : (i == 2 ? v[2] : v[3]);
}

// a set-up camera ray waiting for the warp (k_warp sets up 32 rays at once)
struct RaySetup {
    double d[3], inv[3];
    double rho, tmin, tmax, a, b;  // jitter, clipped range (iso-bounded), root box interval
    int64_t out, slot;
};

// per-ray axis data in shared memory (one copy per warp)
struct RayAxes {
    double o[3], inv[3];
    int sgn[3];  // sign of d: -1, 0, +1
};

// Split the ray interval [tn, tf] of a k-d cell at plane `ph` (half units) on
// `axis` into the intervals of its left (below) and right sides, exactly as
// kd_next classifies children: tp >= tf -> near side only, tp <= tn -> far
// side only, else near [tn, tp] and far [tp, tf]; with d_axis == 0 only the
// side holding the origin (half-open).  An empty side gets lo >= hi.  Returns
// true when the left side is the near one.
__device__ __forceinline__ bool split_sides(const RayAxes& R, int axis, int ph, double tn, double tf, double lo[2],
                                            double hi[2]) {
    const double p = (double)ph * 0.5;
    const double oa = R.o[axis], ia = R.inv[axis];
    const int sg = R.sgn[axis];
    const double tp = (p - oa) * ia;
    const double cut_lo = fmax(tn, tp), cut_hi = fmin(tf, tp);
    if (sg > 0) {
        lo[0] = tn; hi[0] = cut_hi; lo[1] = cut_lo; hi[1] = tf;
    } else if (sg < 0) {
        lo[0] = cut_lo; hi[0] = tf; lo[1] = tn; hi[1] = cut_hi;
    } else {
        const bool below = oa < p;
        lo[0] = tn; hi[0] = below ? tf : tn; lo[1] = tn; hi[1] = below ? tn : tf;
    }
    return sg >= 0;
}

__device__ __forceinline__ int kd4_child(const Kd4Node& nd, int s) {
    return s < 2 ? (s == 0 ? nd.child[0] : nd.child[1]) : (s == 2 ? nd.child[2] : nd.child[3]);
}

// lattice of one region visit (R/render.py:404-418): the samples are the k in
// [kf, ke) with t_in < dt*(k+rho) < t_out, plus the final one at t_out.
__device__ __forceinline__ void lattice(const MarchConst& M, int lev, double ci, double co, double rho, double& kf,
                                        int& cnt) {
    const double dt = M.lv_dt[lev];
    double k = floor(div_dt(M, lev, ci) - rho) + 1.0;
    for (;;) {  // skipped lattice points (tk <= t_in): at most a couple
        const double tk = dt * (k + rho);
        if (tk >= co || tk > ci) break;
        k += 1.0;
    }
    kf = k;
    double ke = floor(div_dt(M, lev, co) - rho);
    if (ke < kf) ke = kf;
    while (ke > kf && dt * ((ke - 1.0) + rho) >= co) ke -= 1.0;
    while (dt * (ke + rho) < co) ke += 1.0;
    cnt = (int)(ke - kf) + 1;
}

// ---------------------------------------------------------------------------
// (Round 2 measured a persistent lane-refill form of both passes — one walk
// step per loop iteration, idle lanes taking the next ray by a warp-aggregated
// atomic — against these one-ray-per-thread kernels: orbit-mean C3 0.905 vs
// 0.898 ms, C2 6.32 vs 6.04, C5 3.47 vs 3.34.  Refilled lanes lose the screen
// coherence of a warp's 32 neighbouring rays, and the block scheduler already
// balances the short blocks.  A warp-cooperative pass 2 — one warp per cut ray
// continuing with k_warp's ordered frontier, 32 node loads in flight — lost as
// well: C2 6.55 vs 6.05 ms, C5 3.91 vs 3.35 (commit 3643681, reverted): most
// frontiers are narrow, so the warp's lanes idle in each expansion step.)
// k_walk: the traversal half of the frame, one thread per ray.  Each thread
// walks the Kd4 tree front to back with a private stack and lists the active
// leaf regions its ray meets, in r_in order, culled only by [t_min, t_max]
// (no restart chain, no early termination: k_warp applies both exactly while
// it consumes the list).  A ray with more than leaf_cap leaves is marked
// truncated and k_warp continues it with the warp frontier from the root.
// Many small independent walks at high occupancy replace the warp frontier's
// narrow expansion steps (a ray's k-d subtree rarely fills 32 lanes).

constexpr int kWalkStack = 100;  // >= 3 x (Kd4 depth <= kKdStack / 2 + 1)
constexpr int kLeafCountMask = 0x0fffffff;
constexpr int kLeafTruncated = 0x40000000;
constexpr int kLeafHeavy = 0x20000000;  // > kShortSamples estimated samples (not for k_short)
constexpr int kLeafTauStop = 0x10000000; // truncated by the opacity minorant (probably terminated)

// pixel of a ray that meets no active region: transparent, or the iso colour
__device__ __forceinline__ void write_empty_pixel(const RenderArgs& A, int64_t slot, int64_t out, bool clip_ok) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    if (A.M.iso_on && clip_ok) {
        const double f = A.iso_shade[slot];
        if (f >= 0.0) {
            acc[0] = A.M.iso_rgb[0] * f;
            acc[1] = A.M.iso_rgb[1] * f;
            acc[2] = A.M.iso_rgb[2] * f;
            acc[3] = 1.0;
        }
    }
    write_pixel(A, out, acc, 0, 0);
}

// The ordered rest of a truncated walk — the pending entry (if any) followed by
// the stack from top to bottom — is exactly a warp-frontier list (disjoint
// subtrees in ray order, conservative float intervals): k_warp resumes from it
// instead of re-descending from the root.  More than kResume entries: none
// saved (k_warp restarts at the root, which is exact as well).
constexpr int kNoEntry = 0x7fffffff;
__device__ __forceinline__ void save_resume(const RenderArgs& A, int64_t slot, int code, double tn, double tf,
                                            const int* st_code, const float* st_tn, const float* st_tf, int sp_n) {
    int32_t* __restrict__ res = A.resume + slot * (int64_t)(1 + 3 * kResume);
    const int m = (code != kNoEntry ? 1 : 0) + sp_n;
    if (m > kResume) {
        res[0] = -1;
        return;
    }
    res[0] = m;
    int k = 0;
    if (code != kNoEntry) {
        res[1 + 3 * k] = code;
        res[2 + 3 * k] = __float_as_int(__double2float_rd(tn));
        res[3 + 3 * k] = __float_as_int(__double2float_ru(tf));
        k++;
    }
    for (int q = sp_n - 1; q >= 0; q--, k++) {
        res[1 + 3 * k] = st_code[q];
        res[2 + 3 * k] = __float_as_int(st_tn[q]);
        res[3 + 3 * k] = __float_as_int(st_tf[q]);
    }
}

// Rays that can meet an active region (root box hit after clipping) -> flag
// (hit_select lists them); the others get their (empty / iso-coloured) pixel
// here and are done.
__global__ void __launch_bounds__(kWalkThreads) k_classify(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= n_slots) return;
    const SceneView& S = A.S;
    const SlotPix spx = slot_pixel(A, slot);
    bool cand = false;
    if (spx.live) {
        Ray r;
        pixel_ray(A, spx.x, spx.y, r);
        double tmin = 0.0, tmax = kTFar;
        clip_ray(A.M, r, tmin, tmax);
        const bool clip_ok = tmin < tmax;
        double a = 0.0, b = -1.0;
        slab_h(S.root_lo, S.root_hi, r, a, b);
        cand = clip_ok && S.n_kd > 0 && a <= b && A.wflags[0];
        if (A.walk_iso) {  // iso phase: default "no hit" (t_end = clip end, no shade)
            A.iso_tend[slot] = tmax;
            A.iso_shade[slot] = -1.0;
        } else if (!cand) {
            write_empty_pixel(A, slot, spx.out, clip_ok);
        }
    } else if (A.walk_iso) {
        A.iso_tend[slot] = -1.0;
        A.iso_shade[slot] = -1.0;
    }
    A.leaf_count[slot] = cand ? -1 : 0;
}

// walk the candidate rays (hit_list[0, n)), one thread each; a walk lists at
// most leaf_cap leaves (long walks are latency chains: k_warp continues those
// rays with its parallel frontier)
// The walk itself (front to back over the Kd4 tree from `code` with the
// ordered stack st_*[0, sp_n)), listing leaves into out[count..cap); on a stop
// it sets `flags` and saves the ordered remainder for k_warp.
__device__ __forceinline__ void walk_leaves(const RenderArgs& A, int64_t slot, const Ray& r, const int sg[3],
                                            double tmin, double tmax, int code, double tn, double tf, int* st_code,
                                            float* st_tn, float* st_tf, int sp_n, int32_t* __restrict__ out,
                                            int& count, int& flags, int cap, float& est) {
    const SceneView& S = A.S;
    const float spc = (float)A.M.spc, tau_stop = A.walk_tau_stop;
    float tau = 0.f;
    for (;;) {
        if (code <= -2) {  // a leaf: list it
            if (count == cap) {  // resume from this leaf
                flags = kLeafTruncated;
                save_resume(A, slot, code, tn, tf, st_code, st_tn, st_tf, sp_n);
                break;
            }
            const int rid = -2 - code;
            out[count++] = rid;
            if (A.short_list && count <= A.short_leaves && est <= A.short_samples)  // samples ~ len/dt + 1
                est += (float)((tf - tn) / A.M.lv_dt[S.rec[rid].meta >> 24]) + 1.f;
            if (A.wqmin) {  // early-stop heuristic: opacity surely past `early` (k_warp verifies)
                tau += __ldg(A.wqmin + rid) * (float)(tf - tn) * spc;
                if (tau > tau_stop) {
                    flags = kLeafTruncated | kLeafTauStop;
                    save_resume(A, slot, kNoEntry, 0.0, 0.0, st_code, st_tn, st_tf, sp_n);
                    break;
                }
            }
        } else {
            // expand the Kd4 node (same classification as kd_next / k_warp)
            const Kd4Node nd = S.kd4[code];
            const uint32_t msk = A.wmask4[code];
            int oc[4];
            double olo[4], ohi[4];
            int no = 0;
            int hs0 = 0, hs1 = 0, nh = 1;
            double hn0 = tn, hf0 = tf, hn1 = 0.0, hf1 = 0.0;
            {
                const int ax = nd.axes & 3;
                const double p = (double)nd.plane[0] * 0.5;
                const double oa = sel3(ax, r.o);
                const int sa = ax == 0 ? sg[0] : (ax == 1 ? sg[1] : sg[2]);
                if (sa == 0) {
                    hs0 = oa < p ? 0 : 1;
                } else {
                    const double tp = (p - oa) * sel3(ax, r.inv);
                    const int ns_ = sa > 0 ? 0 : 1;
                    if (tp >= tf) hs0 = ns_;
                    else if (tp <= tn) hs0 = 1 - ns_;
                    else { hs0 = ns_; hf0 = tp; hs1 = 1 - ns_; hn1 = tp; hf1 = tf; nh = 2; }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                if (h < nh) {
                    const int sd = h ? hs1 : hs0;
                    const double hn = h ? hn1 : hn0, hf = h ? hf1 : hf0;
                    const int ax = (nd.axes >> (2 + 2 * sd)) & 3;
                    int s0 = 2 * sd, s1 = -1;
                    double a0 = hn, b0 = hf, a1 = 0.0, b1 = 0.0;
                    if (ax != 3) {
                        const double p = (double)(sd ? nd.plane[2] : nd.plane[1]) * 0.5;
                        const double oa = sel3(ax, r.o);
                        const int sa = ax == 0 ? sg[0] : (ax == 1 ? sg[1] : sg[2]);
                        if (sa == 0) {
                            s0 = 2 * sd + (oa < p ? 0 : 1);
                        } else {
                            const double tp = (p - oa) * sel3(ax, r.inv);
                            const int nq = sa > 0 ? 0 : 1;
                            if (tp >= b0) s0 = 2 * sd + nq;
                            else if (tp <= a0) s0 = 2 * sd + 1 - nq;
                            else { s0 = 2 * sd + nq; b0 = tp; s1 = 2 * sd + 1 - nq; a1 = tp; b1 = hf; }
                        }
                    }
                    if (((msk >> s0) & 1) && b0 > tmin && a0 < tmax) {
                        oc[no] = kd4_child(nd, s0); olo[no] = a0; ohi[no] = b0; no++;
                    }
                    if (s1 >= 0 && ((msk >> s1) & 1) && b1 > tmin && a1 < tmax) {
                        oc[no] = kd4_child(nd, s1); olo[no] = a1; ohi[no] = b1; no++;
                    }
                }
            }
            if (no > 0) {  // continue with the nearest child, stack the others farthest-first
                if (sp_n + no - 1 > kWalkStack) __trap();  // depth-bounded: <= 3 per Kd4 level
                for (int c = no - 1; c >= 1; c--) {
                    st_code[sp_n] = oc[c];
                    st_tn[sp_n] = __double2float_rd(olo[c]);
                    st_tf[sp_n] = __double2float_ru(ohi[c]);
                    sp_n++;
                }
                code = oc[0];
                tn = olo[0];
                tf = ohi[0];
                continue;
            }
        }
        if (sp_n == 0) break;
        --sp_n;
        code = st_code[sp_n];
        tn = (double)st_tn[sp_n];
        tf = (double)st_tf[sp_n];
    }
}

// route of a walked ray: short (complete list of <= short_leaves leaves, few
// samples) -> k_short, the rest -> k_warp / k_iso_warp; walks cut at the
// pass-1 cap (not by the opacity minorant) also -> k_walk2
__device__ __forceinline__ void route_of(const RenderArgs& A, int v, bool& is_short, bool& is_long, bool& is_cut) {
    const bool any = v != 0;
    is_short = A.short_list && any && !(v & (kLeafTruncated | kLeafHeavy)) && (v & kLeafCountMask) <= A.short_leaves;
    is_long = any && !is_short;
    is_cut = A.cut_list && (v & kLeafTruncated) && (A.cut_tau || !(v & kLeafTauStop));
}

__global__ void __launch_bounds__(kWalkThreads) k_walk(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    const SceneView& S = A.S;
    const int64_t n_cand = (int64_t)A.walk_counter[3];
    // Pass 1 lists at most walk_cap1 leaves per ray: a few very long walks (latency
    // chains of node loads) would otherwise set the kernel's length; k_walk2
    // continues the cap-truncated walks when there are many of them.
    const int cap = A.walk_cap1;
    if (blockIdx.x * (int64_t)blockDim.x >= n_cand) return;
    bool is_short = false, is_long = false, is_cut = false;
    {
        const int64_t ci = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
        if (ci >= n_cand) goto route;
        const int64_t slot = A.hit_list[ci];
        int count = 0, flags = 0;
        const SlotPix spx = slot_pixel(A, slot);
        if (spx.live) {
            Ray r;
            pixel_ray(A, spx.x, spx.y, r);
            double tmin = 0.0, tmax = kTFar;
            clip_ray(A.M, r, tmin, tmax);
            const bool clip_ok = tmin < tmax;
            if (clip_ok && A.M.iso_on && !A.walk_iso) tmax = A.iso_tend[slot];
            double a = 0.0, b = -1.0;
            slab_h(S.root_lo, S.root_hi, r, a, b);
            if (clip_ok && S.n_kd > 0 && a <= b && A.wflags[0]) {
                int st_code[kWalkStack];
                float st_tn[kWalkStack], st_tf[kWalkStack];
                int sg[3];
                for (int q = 0; q < 3; q++) sg[q] = r.d[q] > 0.0 ? 1 : (r.d[q] < 0.0 ? -1 : 0);
                float est = 0.f;
                walk_leaves(A, slot, r, sg, tmin, tmax, S.n_kd4 > 0 ? 0 : -2 - (S.kd[0].a >> 2), a, b, st_code, st_tn,
                            st_tf, 0, A.leaves + slot * (int64_t)A.leaf_cap, count, flags, cap, est);
                if (est > A.short_samples) flags |= kLeafHeavy;
            }
            A.leaf_count[slot] = count | flags;
            if (count == 0 && !flags && !A.walk_iso) write_empty_pixel(A, slot, spx.out, true);  // no active region
        } else {
            A.leaf_count[slot] = 0;
        }
        route_of(A, count | flags, is_short, is_long, is_cut);
    }
route:
    // per-block route counts for k_route (block resources are held until the
    // slowest walk of the block ends anyway, so the barrier costs nothing)
    const int ns = __syncthreads_count(is_short), nl = __syncthreads_count(is_long),
              nc = __syncthreads_count(is_cut);
    if (threadIdx.x == 0) {
        A.blk_counts[3 * blockIdx.x] = ns;
        A.blk_counts[3 * blockIdx.x + 1] = nl;
        A.blk_counts[3 * blockIdx.x + 2] = nc;
    }
    (void)n_slots;
}

// After k_walk: the short / long / cut lists in hit-list (screen) order.  Block b
// takes the hits of k_walk's block b, sums the route counts of the blocks
// before it, ranks its rays with ballots and writes them; the last block
// publishes the list lengths.  (Order matters for speed, not results: lists in
// walk-completion order cost C3 16 %, C2 8 % in k_warp / k_short locality.)
constexpr int kRouteSub = 4;  // k_walk blocks (128 hits each) per k_route block

__global__ void __launch_bounds__(kWalkThreads) k_route(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    __shared__ int s_sum[3][kWalkThreads / 32];
    __shared__ int s_w[3][kWalkThreads / 32];
    const int64_t n_cand = (int64_t)A.walk_counter[3];
    const int64_t nb = (n_cand + kWalkThreads - 1) / kWalkThreads;
    const int64_t bfirst = blockIdx.x * (int64_t)kRouteSub;
    if (bfirst >= nb) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int p0 = 0, p1 = 0, p2 = 0;  // route counts of the k_walk blocks before this one's first
    for (int64_t j = threadIdx.x; j < bfirst; j += blockDim.x) {
        p0 += A.blk_counts[3 * j];
        p1 += A.blk_counts[3 * j + 1];
        p2 += A.blk_counts[3 * j + 2];
    }
    for (int o = 16; o > 0; o >>= 1) {
        p0 += __shfl_xor_sync(0xffffffffu, p0, o);
        p1 += __shfl_xor_sync(0xffffffffu, p1, o);
        p2 += __shfl_xor_sync(0xffffffffu, p2, o);
    }
    if (lane == 0) { s_sum[0][wid] = p0; s_sum[1][wid] = p1; s_sum[2][wid] = p2; }
    __syncthreads();
    int b0 = 0, b1 = 0, b2 = 0;  // list offsets of the current 128 hits
#pragma unroll
    for (int w = 0; w < kWalkThreads / 32; w++) { b0 += s_sum[0][w]; b1 += s_sum[1][w]; b2 += s_sum[2][w]; }
    const unsigned lt = (1u << lane) - 1u;
    for (int sub = 0; sub < kRouteSub; sub++) {
        const int64_t bb = bfirst + sub;
        if (bb >= nb) break;  // uniform over the block
        const int64_t ci = bb * kWalkThreads + threadIdx.x;
        bool is_short = false, is_long = false, is_cut = false;
        int64_t slot = 0;
        if (ci < n_cand) {
            slot = A.hit_list[ci];
            route_of(A, A.leaf_count[slot], is_short, is_long, is_cut);
        }
        const unsigned ms = __ballot_sync(0xffffffffu, is_short), ml = __ballot_sync(0xffffffffu, is_long),
                       mc = __ballot_sync(0xffffffffu, is_cut);
        __syncthreads();  // the previous round's s_w reads are done
        if (lane == 0) { s_w[0][wid] = __popc(ms); s_w[1][wid] = __popc(ml); s_w[2][wid] = __popc(mc); }
        __syncthreads();
        int w0 = 0, w1 = 0, w2 = 0, t0 = 0, t1 = 0, t2 = 0;
#pragma unroll
        for (int w = 0; w < kWalkThreads / 32; w++) {
            if (w < wid) { w0 += s_w[0][w]; w1 += s_w[1][w]; w2 += s_w[2][w]; }
            t0 += s_w[0][w]; t1 += s_w[1][w]; t2 += s_w[2][w];
        }
        if (is_short) A.short_list[b0 + w0 + __popc(ms & lt)] = (int32_t)slot;
        if (is_long) A.long_list[b1 + w1 + __popc(ml & lt)] = (int32_t)slot;
        if (is_cut) A.cut_list[b2 + w2 + __popc(mc & lt)] = (int32_t)slot;
        if (A.any_list && (is_short || is_long))  // short + long merged, in hit order
            A.any_list[b0 + b1 + w0 + w1 + __popc((ms | ml) & lt)] = (int32_t)slot;
        b0 += t0;
        b1 += t1;
        b2 += t2;
        if (bb == nb - 1 && threadIdx.x == 0) {  // the last 128 hits: the list lengths
            A.walk_counter[0] = (unsigned long long)b0;
            A.walk_counter[1] = (unsigned long long)b1;
            A.walk_counter[2] = (unsigned long long)b2;
            A.walk_counter[4] = (unsigned long long)(b0 + b1);
        }
    }
    (void)n_slots;
}

// Pass 2: continue the walks pass 1 cut at walk_cap1 (not those stopped by the
// opacity minorant) up to leaf_cap, from their saved ordered remainder — only
// when there are at least walk2_min of them (decided on the device): many long
// rays (C2, C5) are cheaper here than in k_warp's frontier; a few (C3) are not.

__global__ void __launch_bounds__(kWalkThreads) k_walk2(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    const int64_t n_cut = (int64_t)A.walk_counter[2];
    if (n_cut < A.walk2_min) return;
    const int64_t ci = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (ci >= n_cut) return;
    const int64_t slot = A.cut_list[ci];
    int32_t* res = A.resume + slot * (int64_t)(1 + 3 * kResume);
    const int m = res[0];
    if (m <= 0) return;  // remainder not saved: k_warp restarts at the root
    const SlotPix spx = slot_pixel(A, slot);
    Ray r;
    pixel_ray(A, spx.x, spx.y, r);
    double tmin = 0.0, tmax = kTFar;
    clip_ray(A.M, r, tmin, tmax);
    if (A.M.iso_on && !A.walk_iso) tmax = A.iso_tend[slot];
    int st_code[kWalkStack];
    float st_tn[kWalkStack], st_tf[kWalkStack];
    int sp_n = 0;
    for (int k = m - 1; k >= 1; k--, sp_n++) {  // entries 1.. on the stack, entry 1 on top
        st_code[sp_n] = res[1 + 3 * k];
        st_tn[sp_n] = __int_as_float(res[2 + 3 * k]);
        st_tf[sp_n] = __int_as_float(res[3 + 3 * k]);
    }
    int sg[3];
    for (int q = 0; q < 3; q++) sg[q] = r.d[q] > 0.0 ? 1 : (r.d[q] < 0.0 ? -1 : 0);
    const int lraw = A.leaf_count[slot];
    int count = lraw & kLeafCountMask, flags = lraw & kLeafHeavy;
    float est = INFINITY;
    walk_leaves(A, slot, r, sg, tmin, tmax, res[1], (double)__int_as_float(res[2]), (double)__int_as_float(res[3]),
                st_code, st_tn, st_tf, sp_n, A.leaves + slot * (int64_t)A.leaf_cap, count, flags, A.leaf_cap, est);
    A.leaf_count[slot] = count | flags;
    (void)n_slots;
}
template <bool COUNT>
__global__ void __launch_bounds__(kWarpThreads) k_iso_warp(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const SceneView& S = A.S;
    const int64_t n_cand = (int64_t)A.walk_counter[1];
    const double iso = A.M.iso_value;
    unsigned long long bytes = 0;
    for (;;) {
        unsigned long long c = 0;
        if (lane == 0) c = atomicAdd(A.work_counter, 1ull);
        c = __shfl_sync(FULL, c, 0);
        if ((int64_t)c >= n_cand) break;
        const int64_t slot = A.long_list[c];
        const SlotPix sp = slot_pixel(A, slot);
        Ray r;
        pixel_ray(A, sp.x, sp.y, r);
        const double rho = rho_hash((uint64_t)sp.pix, A.M.seed);
        double tmin = 0.0, tmax = kTFar;
        clip_ray(A.M, r, tmin, tmax);
        const int lraw = A.leaf_count[slot];
        const int32_t* __restrict__ list = A.leaves + slot * (int64_t)A.leaf_cap;
        const int lcount = lraw & kLeafCountMask;
        const bool ltrunc = (lraw & kLeafTruncated) != 0;
        int lpos = 0;
        bool walking = false;
        KdWalk w;
        double t = tmin;
        for (;;) {
            // next region (all lanes compute the same): the list, then the k-d walk
            int rid = -1;
            double ci = 0.0, co = 0.0;
            bool got = false;
            if (!walking) {
                while (lpos < lcount) {
                    const int reg = list[lpos++];
                    const RegionRec q = S.rec[reg];
                    double r_in, r_out;
                    slab_h(q.lo, q.hi, r, r_in, r_out);
                    const double a = r_in > t ? r_in : t, b = r_out < tmax ? r_out : tmax;
                    if (a < b) {
                        rid = reg; ci = a; co = b; got = true;
                        break;
                    }
                }
                if (!got && ltrunc) {
                    walking = true;
                    kd_begin(S, r, w);
                }
            }
            if (walking) got = kd_next(S, A.iflags, r, w, t, tmax, rid, ci, co);
            if (!got) break;
            const RegionRec rr = S.rec[rid];
            const int nids = rr.meta & 0xffffff;
            const int32_t* ids = S.rids + rr.ids_begin;
            if (COUNT && lane == 0) bytes += 32 + 4 * (unsigned long long)nids;
            const double dt = A.M.lv_dt[rr.meta >> 24];
            double kf;
            int cnt;
            lattice(A.M, rr.meta >> 24, ci, co, rho, kf, cnt);  // points p_0 = t_in, p_1..p_cnt (p_cnt = t_out)
            double carry_f = 0.0, carry_t = ci;
            bool carry_ok = false, hit = false;
            double th = 0.0, g[3] = {0.0, 0.0, 0.0};
            for (int base = 0; base <= cnt && !hit; base += 32) {
                const int i = base + lane;
                const bool act = i <= cnt;
                const double ti = i == 0 ? ci : (i >= cnt ? co : dt * ((kf + (double)(i - 1)) + rho));
                bool ok = false;
                double f = 0.0;
                if (act) {
                    Accum Q;
                    gather<false>(S, ids, nids, r.o[0] + ti * r.d[0], r.o[1] + ti * r.d[1], r.o[2] + ti * r.d[2], Q);
                    ok = Q.den > kEpsWeight;
                    f = ok ? Q.num / Q.den - iso : 0.0;
                    if (COUNT) bytes += 16 * (unsigned long long)nids + 4 * (unsigned long long)Q.n_nz;
                }
                double pf = __shfl_up_sync(FULL, f, 1), pt = __shfl_up_sync(FULL, ti, 1);
                bool pok = __shfl_up_sync(FULL, (int)ok, 1) != 0;
                if (lane == 0) { pf = carry_f; pt = carry_t; pok = carry_ok; }
                const bool change = act && i >= 1 && pok && ok && ((pf <= 0.0 && f >= 0.0) || (pf >= 0.0 && f <= 0.0)) &&
                                    !(pf == 0.0 && f == 0.0);
                const unsigned m = __ballot_sync(FULL, change);
                if (m) {
                    const int j = __ffs(m) - 1;
                    if (COUNT) {  // evaluations after the first change were not made by the reference
                        const int lastv = min(31, cnt - base);
                        if (lane > j && lane <= lastv) bytes -= 16 * (unsigned long long)nids;  // n_nz part below
                    }
                    double lo_t = __shfl_sync(FULL, pt, j), hi_t = __shfl_sync(FULL, ti, j);
                    double flo = __shfl_sync(FULL, pf, j);
                    for (int it = 0; it < 16; it++) {  // the reference's bisection, every lane in step
                        const double mid = 0.5 * (lo_t + hi_t);
                        Accum Q;
                        gather<false>(S, ids, nids, r.o[0] + mid * r.d[0], r.o[1] + mid * r.d[1], r.o[2] + mid * r.d[2],
                                      Q);
                        if (COUNT && lane == 0) bytes += 16 * (unsigned long long)nids + 4 * (unsigned long long)Q.n_nz;
                        const double fm = Q.den > kEpsWeight ? Q.num / Q.den - iso : 0.0;
                        if ((flo <= 0.0 && fm <= 0.0) || (flo >= 0.0 && fm >= 0.0)) { lo_t = mid; flo = fm; }
                        else hi_t = mid;
                    }
                    th = 0.5 * (lo_t + hi_t);
                    Accum Q;
                    gather<true>(S, ids, nids, r.o[0] + th * r.d[0], r.o[1] + th * r.d[1], r.o[2] + th * r.d[2], Q);
                    if (Q.den > kEpsWeight) {
                        const double d2 = Q.den * Q.den;
                        for (int a = 0; a < 3; a++) g[a] = (Q.dn[a] * Q.den - Q.gnum * Q.dd[a]) / d2;
                    }
                    hit = true;
                    break;
                }
                const int lastv = min(31, cnt - base);
                carry_f = __shfl_sync(FULL, f, lastv);
                carry_t = __shfl_sync(FULL, ti, lastv);
                carry_ok = __shfl_sync(FULL, (int)ok, lastv) != 0;
            }
            if (hit) {
                if (lane == 0) {
                    A.iso_tend[slot] = th;
                    A.iso_shade[slot] = shade_factor(g, r);
                }
                break;
            }
            t = restart_t(co);
            if (t >= tmax) break;
        }
    }
    if (COUNT) {
        for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(FULL, bytes, o);
        if (lane == 0 && bytes) atomicAdd(&A.stats[2], bytes);
    }
    (void)n_slots;
}

// k_short: one thread per short ray (C3: 87 % of the rays that meet an active
// region list 1-8 leaves and take a handful of samples, which would leave most
// lanes of a warp-per-ray chunk idle).  The thread runs the reference's
// _volume_ray loop over its leaf list verbatim (R/render.py:380-453: exact
// restart chain, lattice, sequential front-to-back compositing, early
// termination) with the frame kernel's reconstruction and shading.
// One short ray by one thread: the reference's _volume_ray loop
// (R/render.py:380-453) over the ray's complete leaf list — exact restart chain,
// lattice, sequential front-to-back compositing, early termination — with the
// frame kernel's reconstruction and shading.  Used by k_short and by k_warp's
// short-ray phase.
template <int GRAD, bool ISO, bool COUNT>
__device__ __forceinline__ void short_ray(const RenderArgs& A, const double* __restrict__ s_tf, int64_t slot,
                                          unsigned long long& my_reg, unsigned long long& my_smp,
                                          unsigned long long& my_bytes) {
    const SceneView& S = A.S;
    const SlotPix sp = slot_pixel(A, slot);
    Ray r;
    pixel_ray(A, sp.x, sp.y, r);
    const double rho = rho_hash((uint64_t)sp.pix, A.M.seed);
    double tmin = 0.0, tmax = kTFar;
    clip_ray(A.M, r, tmin, tmax);
    if (ISO) tmax = A.iso_tend[slot];
    const int count = A.leaf_count[slot] & kLeafCountMask;
    const int32_t* __restrict__ list = A.leaves + slot * (int64_t)A.leaf_cap;
    double ar = 0.0, ag = 0.0, ab = 0.0, aa = 0.0;
    int nreg = 0, nsmp = 0;
    bool fix = false;
    double t = tmin;
    for (int li = 0; li < count && aa < A.M.early; li++) {
        const int rid = list[li];
        const RegionRec rr = S.rec[rid];
        double r_in, r_out;
        slab_h(rr.lo, rr.hi, r, r_in, r_out);
        const double ci = r_in > t ? r_in : t, co = r_out < tmax ? r_out : tmax;
        if (!(ci < co)) continue;  // not the reference's next hit
        nreg++;
        const int lev = rr.meta >> 24, nids = rr.meta & 0xffffff;
        const int32_t* ids = S.rids + rr.ids_begin;
        if (COUNT) my_bytes += 32 + 4 * (unsigned long long)nids;
        const double dt = A.M.lv_dt[lev];
        double prev = ci, k = floor(div_dt(A.M, lev, ci) - rho) + 1.0;
        bool done = false;
        while (!done) {
            double tk = dt * (k + rho);
            k += 1.0;
            if (tk >= co) { tk = co; done = true; }
            else if (tk <= prev) continue;
            const double sl = tk - prev, mid = 0.5 * (prev + tk);
            prev = tk;
            nsmp++;
            const double px = r.o[0] + mid * r.d[0], py = r.o[1] + mid * r.d[1], pz = r.o[2] + mid * r.d[2];
            FastAccum F;
            gather_shade<GRAD == 1>(S, (int64_t)rr.ids_begin, nids, px, py, pz, F);
            if (COUNT) my_bytes += 16 * (unsigned long long)nids + 4 * (unsigned long long)F.n_nz;
            if (F.den > kEpsWeight) {
                const double v = F.num / F.den;
                double c[4];
                tf_eval_fast(s_tf, A.M.tf_lo, A.M.tf_den, A.M.tf_inv, v, c);
                if (c[3] > 0.0) {
                    const double alpha = opacity_correct(c[3], sl * A.M.lv_is1[lev]);
                    if (GRAD != 0) {
                        double f;
                        if (GRAD == 1) {
                            f = shade_factor_f(F.g, r, v);
                            if (f < 0.0) {  // untrusted FP32 gradient (kNegligibleAlpha: see shade_factor_f)
                                fix = fix || alpha >= kNegligibleAlpha;
                                f = 0.2;
                            }
                        } else {
                            double g[3];
                            int64_t ne = 0;
                            central_gradient(S, A.M.grad_mode, px, py, pz, rid, ids, nids, v, g, &ne);
                            f = shade_factor(g, r);
                        }
                        c[0] *= f; c[1] *= f; c[2] *= f;
                    }
                    const double w = alpha * (1.0 - aa);
                    ar += w * c[0];
                    ag += w * c[1];
                    ab += w * c[2];
                    aa += w;
                    if (aa >= A.M.early) break;
                }
            }
        }
        t = restart_t(co);
        if (t >= tmax) break;
    }
    double acc[4] = {ar, ag, ab, aa};
    if (ISO) {
        const double f = A.iso_shade[slot];
        if (f >= 0.0) {
            const double wgt = 1.0 - acc[3];
            acc[0] += wgt * A.M.iso_rgb[0] * f;
            acc[1] += wgt * A.M.iso_rgb[1] * f;
            acc[2] += wgt * A.M.iso_rgb[2] * f;
            acc[3] = 1.0;
        }
    }
    write_pixel(A, sp.out, acc, nreg, nsmp);
    if (fix && A.fixup_list) A.fixup_list[atomicAdd(A.fixup_count, 1ull)] = (int32_t)slot;
    my_reg += nreg;
    my_smp += nsmp;
}

template <int GRAD, bool ISO, bool COUNT>
__global__ void __launch_bounds__(kWalkThreads) k_short(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    __shared__ double s_tf[1024];
    const int64_t n_short = (int64_t)A.walk_counter[0] < A.short_min ? 0 : (int64_t)A.walk_counter[0];
    if (blockIdx.x * (int64_t)blockDim.x >= n_short) return;  // the grid covers every slot; most blocks idle
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = A.tf[i];
    __syncthreads();
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    unsigned long long my_reg = 0, my_smp = 0, my_bytes = 0;
    if (i < n_short) short_ray<GRAD, ISO, COUNT>(A, s_tf, (int64_t)A.short_list[i], my_reg, my_smp, my_bytes);
    for (int o = 16; o > 0; o >>= 1) {
        my_reg += __shfl_xor_sync(0xffffffffu, my_reg, o);
        my_smp += __shfl_xor_sync(0xffffffffu, my_smp, o);
        if (COUNT) my_bytes += __shfl_xor_sync(0xffffffffu, my_bytes, o);
    }
    if ((threadIdx.x & 31) == 0 && A.stats && (my_reg | my_smp)) {
        atomicAdd(&A.stats[0], my_reg);
        atomicAdd(&A.stats[1], my_smp);
        if (COUNT) atomicAdd(&A.stats[2], my_bytes);
    }
    (void)n_slots;
}

template <int GRAD, bool ISO, bool COUNT, int MINB = kWarpMinBlocks>
__global__ void __launch_bounds__(kWarpThreads, MINB) k_warp(const __grid_constant__ RenderArgs A,
                                                                       int64_t n_slots) {
    __shared__ double s_tf[1024];
    __shared__ int s_code[kWarpsPerBlock][32];
    __shared__ double s_tn[kWarpsPerBlock][32], s_tfar[kWarpsPerBlock][32];
    __shared__ SpillEnt s_stack[kWarpsPerBlock][kWarpStack];
    __shared__ SegQ s_q[kWarpsPerBlock][32];
    __shared__ RayAxes s_ray[kWarpsPerBlock];
    __shared__ RaySetup s_setup[kWarpsPerBlock][32];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = A.tf[i];
    __syncthreads();
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const unsigned lt_mask = (1u << lane) - 1u;
    SpillEnt* __restrict__ stk = s_stack[wid];
    const SceneView& S = A.S;
    const double early = A.M.early;
    unsigned long long tot_reg = 0, tot_smp = 0, tot_bytes = 0;
    long long cyc_chunk = 0, cyc_ray = 0, cyc_short = 0;  // DEBUG_CHUNKS: per-warp clock64 sums
    const long long k_t0 = kDebugChunks ? clock64() : 0;
    // work: the long list, or long + short merged when the short rays are too few for k_short
    const bool merged = A.leaves && (!A.short_list || (int64_t)A.walk_counter[0] < A.short_min);
    const int32_t* __restrict__ work = merged ? A.any_list : A.long_list;
    const int64_t n_work = !A.leaves ? n_slots : (int64_t)A.walk_counter[merged ? 4 : 1];

    for (;;) {
        // ---- 32 rays per grab: every lane sets up one ray (camera ray, jitter,
        //      clip, root box); rays that reach no active region are written at
        //      once, the others are marched one after another by the whole warp
        //      Grab size: guided by default (remaining / (grab_div x warps), clamped
        //      to [1, 32]): big grabs while the list is long, single rays at the end,
        //      where a fixed grab of 8 long rays left one warp working while the rest
        //      idled (tools/ab.py, ms, fixed 8 / guided: C3 1.20 / 0.95, C2 6.53 /
        //      6.49, C5 3.63 / 3.62).
        //      With k_walk's leaf lists the work is its hit list (misses are done).
        unsigned long long b0 = 0;
        int grab = 32;
        if (lane == 0) {
            const long long seen = (long long)*(volatile unsigned long long*)A.work_counter;
            const long long left = (long long)n_work - seen;
            const long long g = left / ((long long)A.grab_div * gridDim.x * kWarpsPerBlock);
            grab = A.grab_fixed > 0 ? A.grab_fixed : (int)max(1ll, min(32ll, g));
            b0 = atomicAdd(A.work_counter, (unsigned long long)grab);
        }
        b0 = __shfl_sync(FULL, b0, 0);
        grab = __shfl_sync(FULL, grab, 0);
        if ((int64_t)b0 >= n_work) break;
        const bool my_in = lane < grab && (int64_t)b0 + lane < n_work;
        const int64_t wi = (int64_t)b0 + lane;
        const int64_t my_slot = !A.leaves ? wi : (my_in ? (int64_t)work[wi] : 0);
        SlotPix msp = slot_pixel(A, my_slot);
        msp.live = msp.live && my_in;
        Ray mr;
        pixel_ray(A, msp.x, msp.y, mr);
        const double my_rho = rho_hash((uint64_t)msp.pix, A.M.seed);
        double my_tmin = 0.0, my_tmax = kTFar;
        clip_ray(A.M, mr, my_tmin, my_tmax);
        const bool my_clip_ok = msp.live && my_tmin < my_tmax;
        if (ISO && my_clip_ok) my_tmax = A.iso_tend[my_slot];
        double my_a = 0.0, my_b = -1.0;
        slab_h(S.root_lo, S.root_hi, mr, my_a, my_b);
        const int my_lraw = (A.leaves && msp.live && my_slot < n_slots) ? A.leaf_count[my_slot] : 1;
        const bool my_has = my_clip_ok && S.n_kd > 0 && my_a <= my_b && A.vflags[0] && my_lraw != 0;
        if (msp.live && !my_has) {
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (ISO && my_clip_ok) {
                const double f = A.iso_shade[my_slot];
                if (f >= 0.0) {
                    acc[0] = A.M.iso_rgb[0] * f;
                    acc[1] = A.M.iso_rgb[1] * f;
                    acc[2] = A.M.iso_rgb[2] * f;
                    acc[3] = 1.0;
                }
            }
            write_pixel(A, msp.out, acc, 0, 0);
        }
        unsigned todo = __ballot_sync(FULL, my_has);  // (also orders the previous batch's reads)
        if (my_has) {  // park the ray in shared memory until its turn
            RaySetup& q = s_setup[wid][lane];
            q.d[0] = mr.d[0]; q.d[1] = mr.d[1]; q.d[2] = mr.d[2];
            q.inv[0] = mr.inv[0]; q.inv[1] = mr.inv[1]; q.inv[2] = mr.inv[2];
            q.rho = my_rho; q.tmin = my_tmin; q.tmax = my_tmax; q.a = my_a; q.b = my_b;
            q.out = msp.out;
            q.slot = my_slot;
        }
        __syncwarp();
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const RaySetup& q = s_setup[wid][src];
            const long long r_t0 = kDebugChunks ? clock64() : 0;
            Ray r;
#pragma unroll
            for (int a = 0; a < 3; a++) {
                r.o[a] = A.pos[a];
                r.d[a] = q.d[a];
                r.inv[a] = q.inv[a];
            }
            const double rho = q.rho, tmin = q.tmin, tmax = q.tmax, root_a = q.a, root_b = q.b;
            const int64_t slot = q.slot;
            const int64_t out_px = q.out;
            double Tr = 1.0, Cr = 0.0, Cg = 0.0, Cb = 0.0;  // transmittance, premultiplied colour
            int nreg = 0, nsmp = 0;
            bool fix = false;  // a sample's FP32 gradient was untrusted (shade_factor_f)
            {
                RayAxes& rs = s_ray[wid];
                __syncwarp();
                if (lane < 3) {
                    const double dl = sel3(lane, r.d);
                    rs.o[lane] = sel3(lane, r.o);
                    rs.inv[lane] = sel3(lane, r.inv);
                    rs.sgn[lane] = dl > 0.0 ? 1 : (dl < 0.0 ? -1 : 0);
                }
                __syncwarp();
                double t = tmin;  // the reference's query start (restart chain)
                // ---- frontier: lane i < n holds list entry i; the rest is on the spill stack
                int n = 0, spn = 0;
                int e_code = -1;
                double e_tn = 0.0, e_tf = 0.0;
                // leaf list of k_walk (list mode) or the frontier from the root
                bool lmode = A.leaves != nullptr;
                int lpos = 0, lcnt = 0;
                bool ltrunc = false;
                const int32_t* __restrict__ lbase = nullptr;
                if (lmode) {
                    const int lraw = A.leaf_count[slot];
                    lcnt = lraw & kLeafCountMask;
                    ltrunc = (lraw & kLeafTruncated) != 0;
                    lbase = A.leaves + slot * (int64_t)A.leaf_cap;
                } else {
                    n = 1;  // the root: Kd4 node 0 when the binary root is interior, else a leaf resolved at once
                    if (lane == 0) {
                        e_code = S.n_kd4 > 0 ? 0 : -2 - (S.kd[0].a >> 2);
                        e_tn = root_a;
                        e_tf = root_b;
                    }
                }
                bool walk = true;
                // ---- segment queue: lane i < nq holds visited region i (in ray order)
                //      and q_P = inclusive prefix of the sample counts; h0 samples of
                //      the queue are already composited
                //      (records in the per-warp shared ring s_q from slot qh on)
                int nq = 0, h0 = 0, tailP = 0, qh = 0;
                int q_P = 0x7fffffff;
                SegQ* __restrict__ ring = s_q[wid];
                for (;;) {
                    const int pending = tailP - h0;
                    if (pending >= 32 || (!walk && pending > 0)) {
                        // ================= one chunk of (up to) 32 samples
                        const long long c_t0 = kDebugChunks ? clock64() : 0;
                        const int m = min(32, pending);
                        if (kDebugChunks && A.dbg && lane == 0) {
                            atomicAdd(A.dbg, 1ull);
                            atomicAdd(A.dbg + 1, (unsigned long long)m);
                        }
                        const int s = h0 + lane;
                        const bool act = lane < m;
                        int sg = 0;  // segment of sample s: #{i : q_P[i] <= s}
#pragma unroll
                        for (int b = 16; b >= 1; b >>= 1) {
                            const int v = __shfl_sync(FULL, q_P, sg + b - 1);
                            if (v <= s) sg += b;
                        }
                        sg = min(sg, 31);
                        const SegQ sq = ring[(qh + sg) & 31];
                        const int s_end = __shfl_sync(FULL, q_P, sg);
                        double Ts = 1.0, Cs0 = 0.0, Cs1 = 0.0, Cs2 = 0.0;
                        unsigned long long my_bytes = 0;
                        const int lev = sq.meta >> 24;
                        const int nids = sq.meta & 0xffffff;
                        double sl = 0.0, px = 0.0, py = 0.0, pz = 0.0;
                        if (act) {
                            const double s_dt = A.M.lv_dt[lev];
                            const int j = s - (s_end - sq.cnt);
                            const double prev = j == 0 ? sq.ci : s_dt * ((sq.kf + (double)(j - 1)) + rho);
                            const double tk = j == sq.cnt - 1 ? sq.co : s_dt * ((sq.kf + (double)j) + rho);
                            sl = tk - prev;
                            const double mid = 0.5 * (prev + tk);
                            px = r.o[0] + mid * r.d[0];
                            py = r.o[1] + mid * r.d[1];
                            pz = r.o[2] + mid * r.d[2];
                        }
                        if (kDebugChunks && A.dbg) {
                            int nn = act ? nids : 0, mx = nn;
                            for (int o = 16; o > 0; o >>= 1) {
                                nn += __shfl_xor_sync(FULL, nn, o);
                                mx = max(mx, __shfl_xor_sync(FULL, mx, o));
                            }
                            if (lane == 0) {
                                atomicAdd(A.dbg + 5, (unsigned long long)nn);
                                atomicAdd(A.dbg + 6, (unsigned long long)mx);
                            }
                        }
                        FastAccum F;
                        if (act) {
                            gather_shade<GRAD == 1>(S, (int64_t)sq.ids, nids, px, py, pz, F);
                        }
                        if (act) {
                            if (COUNT) my_bytes = 16 * (unsigned long long)nids + 4 * (unsigned long long)F.n_nz;
                            if (F.den > kEpsWeight) {
                                const double v = F.num / F.den;
                                double c[4];
                                tf_eval_fast(s_tf, A.M.tf_lo, A.M.tf_den, A.M.tf_inv, v, c);
                                if (c[3] > 0.0) {
                                    const double alpha = opacity_correct(c[3], sl * A.M.lv_is1[lev]);
                                    if (GRAD != 0) {
                                        double f;
                                        if (GRAD == 1) {
                                            f = shade_factor_f(F.g, r, v);
                                            if (f < 0.0) {  // untrusted FP32 gradient (see shade_factor_f)
                                                fix = fix || alpha >= kNegligibleAlpha;
                                                f = 0.2;
                                            }
                                        } else {
                                            double g[3];
                                            int64_t ne = 0;
                                            central_gradient(S, A.M.grad_mode, px, py, pz, sq.rid, S.rids + sq.ids,
                                                             nids, v, g, &ne);
                                            f = shade_factor(g, r);
                                        }
                                        c[0] *= f; c[1] *= f; c[2] *= f;
                                    }
                                    Ts = 1.0 - alpha;
                                    Cs0 = alpha * c[0];
                                    Cs1 = alpha * c[1];
                                    Cs2 = alpha * c[2];
                                }
                            }
                        }
                        // inclusive scan of the front-to-back "over" operator
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const double pT = __shfl_up_sync(FULL, Ts, o);
                            const double p0 = __shfl_up_sync(FULL, Cs0, o), p1 = __shfl_up_sync(FULL, Cs1, o),
                                         p2 = __shfl_up_sync(FULL, Cs2, o);
                            if (lane >= o) {
                                Cs0 = p0 + pT * Cs0;
                                Cs1 = p1 + pT * Cs1;
                                Cs2 = p2 + pT * Cs2;
                                Ts = pT * Ts;
                            }
                        }
                        const unsigned tm = __ballot_sync(FULL, act && 1.0 - Tr * Ts >= early);
                        const int last = tm ? __ffs(tm) - 1 : m - 1;
                        const double lT = __shfl_sync(FULL, Ts, last);
                        const double l0 = __shfl_sync(FULL, Cs0, last), l1 = __shfl_sync(FULL, Cs1, last),
                                     l2 = __shfl_sync(FULL, Cs2, last);
                        Cr += Tr * l0;
                        Cg += Tr * l1;
                        Cb += Tr * l2;
                        Tr *= lT;
                        if (COUNT && lane <= last) tot_bytes += my_bytes;
                        if (tm) {  // early termination (R/render.py:448-449): counters stop here
                            const int sg_last = __shfl_sync(FULL, sg, last);
                            nsmp += last + 1;
                            nreg += sg_last + 1;
                            if (COUNT && lane <= sg_last)
                                tot_bytes += 32 + 4 * (unsigned long long)(ring[(qh + lane) & 31].meta & 0xffffff);
                            if (kDebugChunks) cyc_chunk += clock64() - c_t0;
                            break;
                        }
                        nsmp += m;
                        h0 += m;
                        // drop the fully composited segments from the queue front
                        const int k = __popc(__ballot_sync(FULL, lane < nq && q_P <= h0));
                        if (k > 0) {
                            if (COUNT && lane < k)
                                tot_bytes += 32 + 4 * (unsigned long long)(ring[(qh + lane) & 31].meta & 0xffffff);
                            const int done = __shfl_sync(FULL, q_P, k - 1);
                            q_P = __shfl_down_sync(FULL, q_P, k);
                            nq -= k;
                            q_P = lane < nq ? q_P - done : 0x7fffffff;
                            qh = (qh + k) & 31;
                            h0 -= done;
                            tailP -= done;
                            nreg += k;
                        }
                        if (kDebugChunks) cyc_chunk += clock64() - c_t0;
                        continue;
                    }
                    if (!walk) break;
                    // ================= traversal: the next leaves in ray order come from
                    //      k_walk's per-ray list (exact candidates, culled at t_min only), or,
                    //      for a ray whose list was truncated, from the warp frontier
                    //      restarted at the root (culled at the current t: exact as well)
                    int take = 0, leaf_rid = 0;
                    if (lmode) {
                        if (lpos >= lcnt) {
                            lmode = false;
                            if (!ltrunc) {
                                walk = false;
                                continue;
                            }
                            const int32_t* res = A.resume + slot * (int64_t)(1 + 3 * kResume);
                            const int m = res[0];
                            if (m >= 0) {  // resume k_walk's ordered remainder: lanes take the first 32
                                n = min(m, 32);
                                if (lane < n) {
                                    e_code = res[1 + 3 * lane];
                                    e_tn = (double)__int_as_float(res[2 + 3 * lane]);
                                    e_tf = (double)__int_as_float(res[3 + 3 * lane]);
                                }
                                if (m > 32) {  // the rest to the spill stack, earliest on top
                                    spn = m - 32;
                                    for (int q = lane; q < spn; q += 32) {
                                        const int k = 32 + q;  // list entry k -> stack position spn-1-q
                                        stk[spn - 1 - q] = SpillEnt{res[1 + 3 * k], __int_as_float(res[2 + 3 * k]),
                                                                    __int_as_float(res[3 + 3 * k])};
                                    }
                                }
                                __syncwarp();
                            } else {
                                n = 1;
                                if (lane == 0) {
                                    e_code = S.n_kd4 > 0 ? 0 : -2 - (S.kd[0].a >> 2);
                                    e_tn = root_a;
                                    e_tf = root_b;
                                }
                            }
                            continue;
                        }
                        take = min(lcnt - lpos, 32 - nq);  // nq < 32 here: a full queue holds >= 32 samples
                        if (lane < take) leaf_rid = __ldg(lbase + lpos + lane);
                        lpos += take;
                    } else {
                        if (n < 32 && spn > 0) {  // refill the frontier from the spill stack (earliest on top)
                            const int q = min(32 - n, spn);
                            if (lane >= n && lane < n + q) {
                                const SpillEnt f = stk[spn - 1 - (lane - n)];
                                e_code = f.code;
                                e_tn = (double)f.tn;
                                e_tf = (double)f.tf;
                            }
                            spn -= q;
                            n += q;
                            __syncwarp();
                        }
                        if (n == 0) {
                            walk = false;
                            continue;
                        }
                        if (n == 0) {
                            walk = false;
                            continue;
                        }
                        const unsigned leafm = __ballot_sync(FULL, lane < n && e_code <= -2);
                        const int nl = leafm == FULL ? 32 : __ffs(~leafm) - 1;
                        if (nl == 0) {
                            // ---- expansion step: every unresolved entry is a Kd4 node; it is
                            //      replaced in place by its (up to 4) surviving children, near
                            //      first.  Branch-free: each split turns the entry interval into
                            //      the intervals of its two sides with the same exact slab
                            //      arithmetic as kd_next (an empty side gets lo >= hi).
                            bool actx = lane < n && e_code >= 0;
                            if (spn + 96 > kWarpStack) {  // near the spill limit: expand the first entry only
                                const unsigned um = __ballot_sync(FULL, actx);
                                actx = actx && lane == __ffs(um) - 1;
                            }
                            int oc[4] = {e_code, 0, 0, 0};
                            double otn[4] = {e_tn, 0.0, 0.0, 0.0}, otf[4] = {e_tf, 0.0, 0.0, 0.0};
                            bool ov[4] = {lane < n && !actx, false, false, false};  // a resolved leaf stays in place
                            if (actx) {
                                const Kd4Node nd = S.kd4[e_code];
                                const uint32_t msk = A.vmask4[e_code];
                                // first split: one or two halves, in ray order (kd_next's classification)
                                int hs0 = 0, hs1 = 0, nh = 1;
                                double hn0 = e_tn, hf0 = e_tf, hn1 = 0.0, hf1 = 0.0;
                                {
                                    const int ax = nd.axes & 3;
                                    const double p = (double)nd.plane[0] * 0.5;
                                    const int sg = rs.sgn[ax];
                                    const double oa = rs.o[ax];
                                    if (sg == 0) {
                                        hs0 = oa < p ? 0 : 1;
                                    } else {
                                        const double tp = (p - oa) * rs.inv[ax];
                                        const int ns_ = sg > 0 ? 0 : 1;
                                        if (tp >= e_tf) {
                                            hs0 = ns_;
                                        } else if (tp <= e_tn) {
                                            hs0 = 1 - ns_;
                                        } else {
                                            hs0 = ns_; hf0 = tp;
                                            hs1 = 1 - ns_; hn1 = tp; hf1 = e_tf;
                                            nh = 2;
                                        }
                                    }
                                }
        #pragma unroll
                                for (int h = 0; h < 2; h++) {
                                    if (h < nh) {
                                        const int sd = h ? hs1 : hs0;
                                        const double hn = h ? hn1 : hn0, hf = h ? hf1 : hf0;
                                        const int ax = (nd.axes >> (2 + 2 * sd)) & 3;
                                        int s0 = 2 * sd, s1 = -1;
                                        double a0 = hn, bb0 = hf, a1 = 0.0, bb1 = 0.0;
                                        if (ax != 3) {
                                            const double p = (double)(sd ? nd.plane[2] : nd.plane[1]) * 0.5;
                                            const int sg = rs.sgn[ax];
                                            const double oa = rs.o[ax];
                                            if (sg == 0) {
                                                s0 = 2 * sd + (oa < p ? 0 : 1);
                                            } else {
                                                const double tp = (p - oa) * rs.inv[ax];
                                                const int nqq = sg > 0 ? 0 : 1;
                                                if (tp >= bb0) {
                                                    s0 = 2 * sd + nqq;
                                                } else if (tp <= a0) {
                                                    s0 = 2 * sd + 1 - nqq;
                                                } else {
                                                    s0 = 2 * sd + nqq; bb0 = tp;
                                                    s1 = 2 * sd + 1 - nqq; a1 = tp; bb1 = hf;
                                                }
                                            }
                                        }
                                        // cull: inactive subtree, or entirely before t / after tmax
                                        ov[2 * h] = ((msk >> s0) & 1) && bb0 > t && a0 < tmax;
                                        oc[2 * h] = kd4_child(nd, s0); otn[2 * h] = a0; otf[2 * h] = bb0;
                                        ov[2 * h + 1] = s1 >= 0 && ((msk >> s1) & 1) && bb1 > t && a1 < tmax;
                                        oc[2 * h + 1] = kd4_child(nd, s1 < 0 ? 0 : s1); otn[2 * h + 1] = a1; otf[2 * h + 1] = bb1;
                                    }
                                }
                            }
                            const int cnt = (int)ov[0] + (int)ov[1] + (int)ov[2] + (int)ov[3];
                            const unsigned m1 = __ballot_sync(FULL, cnt & 1), m2 = __ballot_sync(FULL, cnt & 2),
                                           m4 = __ballot_sync(FULL, cnt & 4);
                            const int pos = __popc(m1 & lt_mask) + 2 * __popc(m2 & lt_mask) + 4 * __popc(m4 & lt_mask);
                            const int total = __popc(m1) + 2 * __popc(m2) + 4 * __popc(m4);
                            if (spn + max(0, total - 32) > kWarpStack) __trap();  // cannot happen: see the guard above
                            int p = pos;
        #pragma unroll
                            for (int c = 0; c < 4; c++) {
                                if (ov[c]) {
                                    if (p < 32) {
                                        s_code[wid][p] = oc[c];
                                        s_tn[wid][p] = otn[c];
                                        s_tfar[wid][p] = otf[c];
                                    } else {
                                        SpillEnt& f = stk[spn + (total - 1 - p)];
                                        f.code = oc[c];
                                        f.tn = __double2float_rd(otn[c]);
                                        f.tf = __double2float_ru(otf[c]);
                                    }
                                    p++;
                                }
                            }
                            __syncwarp();
                            if (total > 32) spn += total - 32;
                            n = min(total, 32);
                            if (lane < n) {
                                e_code = s_code[wid][lane];
                                e_tn = s_tn[wid][lane];
                                e_tf = s_tfar[wid][lane];
                            }
                            __syncwarp();
                            continue;
                        }
                        take = min(nl, 32 - nq);
                        leaf_rid = lane < take ? -2 - e_code : 0;
                        // shift the frontier past the consumed leaves
                        if (take < 32) {
                            e_code = __shfl_down_sync(FULL, e_code, take);
                            e_tn = __shfl_down_sync(FULL, e_tn, take);
                            e_tf = __shfl_down_sync(FULL, e_tf, take);
                        }
                        n -= take;
                    }
                    {
                        // ---- consume leading leaves into the segment queue: exact slab,
                        //      restart chain t_i = restart(t_out of the previous visit)
                        const bool isleaf = lane < take;
                        const int rid = isleaf ? leaf_rid : 0;
                        RegionRec rr{};
                        double r_in = INFINITY, r_out = -INFINITY;
                        if (isleaf) {
                            rr = S.rec[rid];
                            slab_h(rr.lo, rr.hi, r, r_in, r_out);
                        }
                        double co = r_out < tmax ? r_out : tmax;
                        const double prev_co = __shfl_up_sync(FULL, co, 1);
                        const double ti = lane == 0 ? t : restart_t(prev_co);
                        double ci = r_in > ti ? r_in : ti;
                        bool ok = isleaf && ci < co;
                        const unsigned lmask = take == 32 ? FULL : ((1u << take) - 1u);
                        unsigned okm = __ballot_sync(FULL, ok);
                        bool stop = false;
                        if (okm != lmask) {
                            // a skipped region (thinner than the restart epsilon, or missed
                            // by the ray): resolve the chain sequentially
                            double tt = t;
                            ok = false;
                            for (int i = 0; i < take; i++) {
                                const double ri = __shfl_sync(FULL, r_in, i), ro = __shfl_sync(FULL, r_out, i);
                                const double a = ri > tt ? ri : tt, b = ro < tmax ? ro : tmax;
                                if (a < b) {
                                    if (lane == i) { ok = true; ci = a; co = b; }
                                    tt = restart_t(b);
                                    if (tt >= tmax) { stop = true; break; }
                                }
                            }
                            okm = __ballot_sync(FULL, ok);
                        }
                        const int ns = __popc(okm);
                        if (stop) walk = false;
                        if (ns == 0) continue;
                        int g_rid = rid, g_ids = rr.ids_begin, g_meta = rr.meta;
                        double g_ci = ci, g_co = co;
                        if (okm != ((ns == 32) ? FULL : ((1u << ns) - 1u))) {
                            // rare: gather the ns visited lanes via shared scratch
                            if (ok) {
                                const int p = __popc(okm & lt_mask);
                                s_code[wid][p] = rid;
                                s_tn[wid][p] = ci;
                                s_tfar[wid][p] = co;
                            }
                            __syncwarp();
                            if (lane < ns) {
                                g_rid = s_code[wid][lane];
                                g_ci = s_tn[wid][lane];
                                g_co = s_tfar[wid][lane];
                                const RegionRec q = S.rec[g_rid];
                                g_ids = q.ids_begin;
                                g_meta = q.meta;
                            }
                            __syncwarp();
                        }
                        double g_kf = 0.0;
                        int g_cnt = 0;
                        if (lane < ns) lattice(A.M, g_meta >> 24, g_ci, g_co, rho, g_kf, g_cnt);
                        int P = g_cnt;
#pragma unroll
                        for (int o = 1; o < 32; o <<= 1) {
                            const int v = __shfl_up_sync(FULL, P, o);
                            if (lane >= o) P += v;
                        }
                        const double t_last = __shfl_sync(FULL, g_co, ns - 1);
                        const int S_new = __shfl_sync(FULL, P, 31);
                        // append: new segment i -> window position nq + i (a ring slot the last
                        // chunk may still have been reading: order the warp's reads first)
                        __syncwarp();
                        if (lane < ns) {
                            SegQ& q = ring[(qh + nq + lane) & 31];
                            q.ci = g_ci; q.co = g_co; q.kf = g_kf;
                            q.ids = g_ids; q.meta = g_meta; q.cnt = g_cnt; q.rid = g_rid;
                        }
                        const int u_P = __shfl_up_sync(FULL, P, nq);
                        if (lane >= nq && lane < nq + ns) q_P = tailP + u_P;
                        __syncwarp();
                        nq += ns;
                        tailP += S_new;
                        t = restart_t(t_last);
                        if (t >= tmax) walk = false;
                        continue;
                    }
                }
            }
            if (lane == 0) {
                double acc[4] = {Cr, Cg, Cb, 1.0 - Tr};
                if (ISO) {
                    const double f = A.iso_shade[slot];
                    if (f >= 0.0) {
                        const double wgt = 1.0 - acc[3];
                        acc[0] += wgt * A.M.iso_rgb[0] * f;
                        acc[1] += wgt * A.M.iso_rgb[1] * f;
                        acc[2] += wgt * A.M.iso_rgb[2] * f;
                        acc[3] = 1.0;
                    }
                }
                write_pixel(A, out_px, acc, nreg, nsmp);
            }
            if (__any_sync(FULL, fix) && lane == 0 && A.fixup_list)
                A.fixup_list[atomicAdd(A.fixup_count, 1ull)] = (int32_t)slot;
            if (kDebugChunks) cyc_ray += clock64() - r_t0;
            if (lane == 0) {
                if (kDebugChunks && A.dbg) {
                    atomicAdd(A.dbg + 2, 1ull);
                    atomicAdd(A.dbg + 3, (unsigned long long)nsmp);
                    atomicAdd(A.dbg + 4, (unsigned long long)nreg);
                }
                tot_reg += nreg;
                tot_smp += nsmp;
            }
        }
    }
    // ---- short-ray phase (k_short fused): one short ray per lane, 32 per grab;
    //      cheap, uniform rays fill the tail of the long-ray phase
    const long long s_t0 = kDebugChunks ? clock64() : 0;
    if (A.fuse_short && A.leaves && !merged) {
        const int64_t n_sh = (int64_t)A.walk_counter[0];
        for (;;) {
            unsigned long long c0 = 0;
            if (lane == 0) c0 = atomicAdd(A.short_counter, 32ull);
            c0 = __shfl_sync(FULL, c0, 0);
            if ((int64_t)c0 >= n_sh) break;
            const int64_t i = (int64_t)c0 + lane;
            if (i < n_sh) short_ray<GRAD, ISO, COUNT>(A, s_tf, (int64_t)A.short_list[i], tot_reg, tot_smp, tot_bytes);
        }
    }
    if (kDebugChunks && A.dbg && lane == 0) {
        cyc_short = clock64() - s_t0;
        atomicAdd(A.dbg + 16, (unsigned long long)cyc_chunk);
        atomicAdd(A.dbg + 17, (unsigned long long)cyc_ray);
        atomicAdd(A.dbg + 18, (unsigned long long)cyc_short);
        atomicAdd(A.dbg + 19, (unsigned long long)(s_t0 - k_t0));
    }
    for (int o = 16; o > 0; o >>= 1) {
        tot_reg += __shfl_xor_sync(FULL, tot_reg, o);
        tot_smp += __shfl_xor_sync(FULL, tot_smp, o);
        if (COUNT) tot_bytes += __shfl_xor_sync(FULL, tot_bytes, o);
    }
    if (lane == 0 && A.stats) {
        atomicAdd(&A.stats[0], tot_reg);
        atomicAdd(&A.stats[1], tot_smp);
        if (COUNT) atomicAdd(&A.stats[2], tot_bytes);
    }
}

// ---------------------------------------------------------------------------
// k_fixup: pixels whose FP32 shading gradient was untrusted (shade_factor_f)
// are re-rendered one thread each with the exact per-pixel path — the
// reference's FP64 gradient sums (volume_ray) — after k_warp.  The counters
// are the same as k_warp's, so the frame stats are not touched.

template <bool ISO>
__global__ void __launch_bounds__(128) k_fixup(const __grid_constant__ RenderArgs A) {
    __shared__ double s_tf[1024];
    const int64_t n = (int64_t)*A.fixup_count;
    if (blockIdx.x * (int64_t)blockDim.x >= n) return;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = A.tf[i];
    __syncthreads();
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t slot = A.fixup_list[q];
        const SlotPix sp = slot_pixel(A, slot);
        RayStats st = {0, 0, 0};
        Ray r;
        pixel_ray(A, sp.x, sp.y, r);
        const double rho = rho_hash((uint64_t)sp.pix, A.M.seed);
        double tmin = 0.0, tmax = kTFar;
        clip_ray(A.M, r, tmin, tmax);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (tmin < tmax) {
            const double t_end = ISO ? A.iso_tend[slot] : tmax;
            volume_ray<1, false>(A.S, A.vflags, A.M, s_tf, r, tmin, t_end, rho, acc, st, nullptr);
            if (ISO && A.iso_shade[slot] >= 0.0) {
                const double f = A.iso_shade[slot];
                const double w = 1.0 - acc[3];
                acc[0] += w * A.M.iso_rgb[0] * f;
                acc[1] += w * A.M.iso_rgb[1] * f;
                acc[2] += w * A.M.iso_rgb[2] * f;
                acc[3] = 1.0;
            }
        }
        write_pixel(A, sp.out, acc, (int)st.regions, (int)st.samples);
    }
}

// ---------------------------------------------------------------------------
// simple tile kernel (one thread per pixel), kept for A/B comparison

template <int GRAD, bool ISO, bool COUNT>
__global__ void __launch_bounds__(kTileW* kTileH) k_render(const __grid_constant__ RenderArgs A) {
    __shared__ double s_tf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = A.tf[i];
    __syncthreads();
    const int64_t slot = (int64_t)blockIdx.x * (kTileW * kTileH) + threadIdx.x;
    const SlotPix sp = slot_pixel(A, slot);
    RayStats st = {0, 0, 0};
    if (sp.live) {
        Ray r;
        pixel_ray(A, sp.x, sp.y, r);
        const double rho = rho_hash((uint64_t)sp.pix, A.M.seed);
        double tmin = 0.0, tmax = kTFar;
        clip_ray(A.M, r, tmin, tmax);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (tmin < tmax) {
            double t_end = ISO ? A.iso_tend[slot] : tmax;
            volume_ray<GRAD, COUNT>(A.S, A.vflags, A.M, s_tf, r, tmin, t_end, rho, acc, st,
                                    A.use_lbvh ? &A.vlb : nullptr);
            if (ISO && A.iso_shade[slot] >= 0.0) {
                const double f = A.iso_shade[slot];
                const double w = 1.0 - acc[3];
                acc[0] += w * A.M.iso_rgb[0] * f;
                acc[1] += w * A.M.iso_rgb[1] * f;
                acc[2] += w * A.M.iso_rgb[2] * f;
                acc[3] = 1.0;
            }
        }
        write_pixel(A, sp.out, acc, (int)st.regions, (int)st.samples);
    }
    unsigned long long v0 = st.regions, v1 = st.samples, v2 = st.bytes;
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    if ((threadIdx.x & 31) == 0 && A.stats) {
        atomicAdd(&A.stats[0], v0);
        atomicAdd(&A.stats[1], v1);
        if (COUNT) atomicAdd(&A.stats[2], v2);
    }
}

// ---------------------------------------------------------------------------
// launch

using RenderFn = void (*)(RenderArgs);
using FrameFn = void (*)(RenderArgs, int64_t);

template <int GRAD, bool ISO>
static RenderFn tile_fn(bool count) {
    return count ? (RenderFn)k_render<GRAD, ISO, true> : (RenderFn)k_render<GRAD, ISO, false>;
}

static int grad_index(int mode) { return mode == 0 ? 0 : (mode == 1 ? 1 : 2); }

template <int GRAD, bool ISO>
static FrameFn warp_fn(bool count) {
    return count ? (FrameFn)k_warp<GRAD, ISO, true> : (FrameFn)k_warp<GRAD, ISO, false>;
}

// slots i in [0, n) with pred(i), in order -> out, count -> *n_out (device)
// flagged rays (leaf_count != 0 after k_classify) -> hit_list in slot (screen)
// order, length -> walk_counter[3].  Screen order keeps neighbouring rays
// together in k_walk / k_warp: a list in arrival order (warp-aggregated atomics
// in k_classify) cost C2 / C3 5-7 %.
struct HasLeaves {
    const int32_t* c;
    __device__ __forceinline__ bool operator()(const int32_t i) const { return c[i] != 0; }
};

static void hit_select(const RenderArgs& A, int64_t n_slots, cudaStream_t s) {
    size_t tb = 0;
    cub::CountingInputIterator<int32_t> it(0);
    XB_CUDA(cub::DeviceSelect::If(nullptr, tb, it, A.hit_list, A.walk_counter + 3, (int)n_slots,
                                  HasLeaves{A.leaf_count}, s));
    void* tmp = nullptr;
    XB_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 16), s));
    XB_CUDA(cub::DeviceSelect::If(tmp, tb, it, A.hit_list, A.walk_counter + 3, (int)n_slots,
                                  HasLeaves{A.leaf_count}, s));
    XB_CUDA(cudaFreeAsync(tmp, s));
}

void launch_render(const RenderArgs& A, int64_t n_tiles_local, bool count, cudaStream_t s) {
    if (n_tiles_local <= 0) return;
    NvtxRange frame_range("xb_render: frame");
    const bool iso = A.M.iso_on != 0;
    const int g = grad_index(A.M.grad_mode);
    const int64_t n_slots = n_tiles_local * kTileW * kTileH;
    if (iso && (!A.leaves || A.kernel != 0)) {  // per-lane iso pass (tile / LBVH / frontier-only paths)
        void* args[] = {(void*)&A, (void*)&n_slots};
        const void* fn = count ? (const void*)k_iso_pass<true> : (const void*)k_iso_pass<false>;
        XB_CUDA(cudaLaunchKernel(fn, dim3(grid_for(n_slots, 128)), dim3(128), args, 0, s));
    } else if (iso) {
        // iso phase through the walk machinery: classify, select, walk the iso set, march
        NvtxRange r_iso("iso phase: classify, select, walk, route, k_iso_warp");
        RenderArgs* Ai = new RenderArgs(A);
        std::unique_ptr<RenderArgs> hold(Ai);
        Ai->walk_iso = 1;
        Ai->wflags = A.iflags;
        Ai->wmask4 = A.imask4;
        Ai->wqmin = nullptr;
        Ai->short_list = nullptr;
        Ai->walk_cap1 = std::min(A.leaf_cap, 16);
        void* iargs[] = {(void*)Ai, (void*)&n_slots};
        Ai->cut_list = nullptr;
        XB_CUDA(cudaLaunchKernel((const void*)k_classify, dim3(grid_for(n_slots, kWalkThreads)), dim3(kWalkThreads),
                                 iargs, 0, s));
        hit_select(*Ai, n_slots, s);
        XB_CUDA(cudaLaunchKernel((const void*)k_walk, dim3(grid_for(n_slots, kWalkThreads)), dim3(kWalkThreads), iargs,
                                 0, s));
        XB_CUDA(cudaLaunchKernel((const void*)k_route, dim3(grid_for(n_slots, kWalkThreads * kRouteSub)),
                                 dim3(kWalkThreads), iargs, 0, s));
        {
            const void* mf = count ? (const void*)k_iso_warp<true> : (const void*)k_iso_warp<false>;
            int dev = 0, sms = 0, per_sm = 0;
            XB_CUDA(cudaGetDevice(&dev));
            XB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mf, kWarpThreads, 0));
            XB_CUDA(cudaLaunchKernel(mf, dim3((unsigned)std::max(1, sms * std::max(per_sm, 1))), dim3(kWarpThreads),
                                     iargs, 0, s));
            // k_warp's ray counter is shared: reset it for the volume phase
            XB_CUDA(cudaMemsetAsync(A.work_counter, 0, sizeof(unsigned long long), s));
        }
        XB_CUDA(cudaMemsetAsync(A.walk_counter, 0, 5 * sizeof(unsigned long long), s));  // volume phase lists
    }
    if (A.kernel == 1) {  // one thread per pixel: LBVH traversal, cell location, tuning.kernel = 1
        RenderFn fn;
        if (g == 0) fn = iso ? tile_fn<0, true>(count) : tile_fn<0, false>(count);
        else if (g == 1) fn = iso ? tile_fn<1, true>(count) : tile_fn<1, false>(count);
        else fn = iso ? tile_fn<2, true>(count) : tile_fn<2, false>(count);
        void* args[] = {(void*)&A};
        XB_CUDA(cudaLaunchKernel((const void*)fn, dim3((unsigned)n_tiles_local), dim3(kTileW * kTileH), args, 0, s));
        return;
    }
    FrameFn fn;
    const int threads = kWarpThreads;
    {
        if (A.leaves) {
            RenderArgs& W = const_cast<RenderArgs&>(A);
            const double e = std::min(A.M.early, 0.999999);
            // walks stop once the opacity minorant passes `early` (opacity >= 1 - e^-tau); a ray that
            // did not terminate there resumes in k_warp, so the margin only trades walk length
            // against resumes (tools/ab.py, ms, margin 2 / 1 / 0 / -1: C5 3.48 / 3.38 / 3.31 / 3.57,
            // C2 6.30 / 6.30 / 6.27 / 6.42, C3 flat)
            W.walk_tau_stop = (float)(-std::log(1.0 - e));
            void* wargs[] = {(void*)&A, (void*)&n_slots};
            NvtxRange r_walk("walk phase: k_classify, hit select, k_walk, k_route, k_walk2");
            XB_CUDA(cudaLaunchKernel((const void*)k_classify, dim3(grid_for(n_slots, kWalkThreads)),
                                     dim3(kWalkThreads), wargs, 0, s));
            hit_select(A, n_slots, s);
            // one thread per candidate (blocks past the device-side count exit at once), then
            // k_route builds the short / long / cut lists
            XB_CUDA(cudaLaunchKernel((const void*)k_walk, dim3(grid_for(n_slots, kWalkThreads)), dim3(kWalkThreads),
                                     wargs, 0, s));
            XB_CUDA(cudaLaunchKernel((const void*)k_route, dim3(grid_for(n_slots, kWalkThreads * kRouteSub)),
                                     dim3(kWalkThreads), wargs, 0, s));
            if (A.cut_list && A.walk_cap1 < A.leaf_cap)  // pass 2 over the cap-cut walks
                XB_CUDA(cudaLaunchKernel((const void*)k_walk2, dim3(grid_for(n_slots, kWalkThreads)),
                                         dim3(kWalkThreads), wargs, 0, s));
            if (A.short_list && !A.fuse_short) {  // short rays -> k_short (when >= short_min of them)
                using ShortFn = void (*)(RenderArgs, int64_t);
                ShortFn sf;
                if (g == 0) sf = iso ? (ShortFn)k_short<0, true, false> : (ShortFn)k_short<0, false, false>;
                else if (g == 1) sf = iso ? (ShortFn)k_short<1, true, false> : (ShortFn)k_short<1, false, false>;
                else sf = iso ? (ShortFn)k_short<2, true, false> : (ShortFn)k_short<2, false, false>;
                if (count) {
                    if (g == 0) sf = iso ? (ShortFn)k_short<0, true, true> : (ShortFn)k_short<0, false, true>;
                    else if (g == 1) sf = iso ? (ShortFn)k_short<1, true, true> : (ShortFn)k_short<1, false, true>;
                    else sf = iso ? (ShortFn)k_short<2, true, true> : (ShortFn)k_short<2, false, true>;
                }
                XB_CUDA(cudaLaunchKernel((const void*)sf, dim3(grid_for(n_slots, kWalkThreads)), dim3(kWalkThreads),
                                         wargs, 0, s));
            }
        }
        if (g == 0) fn = iso ? warp_fn<0, true>(count) : warp_fn<0, false>(count);
        else if (g == 1) fn = iso ? warp_fn<1, true>(count) : warp_fn<1, false>(count);
        else fn = iso ? warp_fn<2, true>(count) : warp_fn<2, false>(count);
    }
    int dev = 0, sms = 0, per_sm = 0;
    XB_CUDA(cudaGetDevice(&dev));
    XB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    size_t dyn = 0;
    XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, threads, dyn));
    const int64_t want = (n_slots * 32 + threads - 1) / threads;  // k_warp: one ray per warp at a time
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), want));
    void* args[] = {(void*)&A, (void*)&n_slots};
    cudaEvent_t* ev = (cudaEvent_t*)A.march_events;
    NvtxRange r_march("march: k_warp");
    if (ev) XB_CUDA(cudaEventRecord(ev[0], s));
    XB_CUDA(cudaLaunchKernel((const void*)fn, dim3((unsigned)blocks), dim3(threads), args, dyn, s));
    if (ev) XB_CUDA(cudaEventRecord(ev[1], s));
    if (A.fixup_list && g == 1 && !count) {  // untrusted FP32 gradients: exact re-render of those pixels
        void* fargs[] = {(void*)&A};
        const void* ff = iso ? (const void*)k_fixup<true> : (const void*)k_fixup<false>;
        XB_CUDA(cudaLaunchKernel(ff, dim3((unsigned)sms), dim3(128), fargs, 0, s));
    }
}

// ---------------------------------------------------------------------------
// ray batch: integrate_ray (R/render.py:613-632) and iso_intersect (635-651)

__global__ void k_rays(const __grid_constant__ RayBatchArgs B) {
    __shared__ double s_tf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = B.tf[i];
    __syncthreads();
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= B.n) return;
    Ray r;
    for (int a = 0; a < 3; a++) {
        r.o[a] = B.o[3 * q + a];
        r.d[a] = B.d[3 * q + a];
        r.inv[a] = 1.0 / r.d[a];
    }
    double tmin = B.t0[q], tmax = B.t1[q];
    const double rho = B.rho[q];
    RayStats st = {0, 0, 0};
    const LbvhView* vl = B.use_lbvh ? &B.vlb : nullptr;
    if (B.mode == 0) {  // volume integration
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        clip_ray(B.M, r, tmin, tmax);
        if (tmin < tmax) {
            switch (B.M.grad_mode) {
                case 0: volume_ray<0, false>(B.S, B.vflags, B.M, s_tf, r, tmin, tmax, rho, acc, st, vl); break;
                case 1: volume_ray<1, false>(B.S, B.vflags, B.M, s_tf, r, tmin, tmax, rho, acc, st, vl); break;
                default: volume_ray<2, false>(B.S, B.vflags, B.M, s_tf, r, tmin, tmax, rho, acc, st, vl); break;
            }
        }
        for (int c = 0; c < 4; c++) B.out[4 * q + c] = acc[c];
        B.counts[2 * q] = st.regions;
        B.counts[2 * q + 1] = st.samples;
    } else {  // iso intersection
        double g[3], th = 0.0;
        const bool hit = iso_ray<false>(B.S, B.iflags, B.M, r, tmin, tmax, rho, th, g, st, B.use_lbvh ? &B.ilb : nullptr);
        B.out[4 * q] = th;
        for (int c = 0; c < 3; c++) B.out[4 * q + 1 + c] = g[c];
        B.counts[2 * q] = hit ? 1 : 0;
        B.counts[2 * q + 1] = 0;
    }
}

void launch_rays(const RayBatchArgs& B, cudaStream_t s) {
    if (B.n <= 0) return;
    void* args[] = {(void*)&B};
    XB_CUDA(cudaLaunchKernel((const void*)k_rays, dim3(grid_for(B.n, 64)), dim3(64), args, 0, s));
}

// ---------------------------------------------------------------------------
// multi-GPU: scatter packed tiles (rank-major gather buffer) into the image

__global__ void k_unpack_tiles(const uchar4* __restrict__ packed, int64_t tiles_per_rank, int world, int tiles_x,
                               int tiles_y, int W, int H, uchar4* __restrict__ img) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t tile_px = kTileW * kTileH;
    const int64_t total = tiles_per_rank * world * tile_px;
    if (q >= total) return;
    const int64_t slot = q / tile_px;
    const int local = (int)(q % tile_px);
    const int rank = (int)(slot / tiles_per_rank);
    const int64_t t_local = slot % tiles_per_rank;
    const int64_t tile = rank + t_local * world;
    if (tile >= (int64_t)tiles_x * tiles_y) return;
    const int x = (int)(tile % tiles_x) * kTileW + local % kTileW;
    const int y = (int)(tile / tiles_x) * kTileH + local / kTileW;
    if (x < W && y < H) img[(int64_t)y * W + x] = packed[q];
}

void launch_unpack(const uchar4* packed, int64_t tiles_per_rank, int world, int tiles_x, int tiles_y, int W, int H,
                   uchar4* img, cudaStream_t s) {
    const int64_t total = tiles_per_rank * world * kTileW * kTileH;
    if (total <= 0) return;
    k_unpack_tiles<<<grid_for(total, 256), 256, 0, s>>>(packed, tiles_per_rank, world, tiles_x, tiles_y, W, H, img);
    check_launch("k_unpack_tiles");
}

}  // namespace xb
