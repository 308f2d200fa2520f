// accel.cu — transfer-function majorants, active region sets, k-d subtree
// flags, point sampling and interval tracing (paper §3.3, §4.1, §5.2).
//
// `build_volume_bvh` / `build_iso_bvh` / `build_all_regions_bvh`
// (R/accel.py:227-247) become: one kernel evaluating the exact FP64
// `max_opacity` (R/accel.py:91-115) or the iso bracket test per region, then a
// bottom-up OR over the k-d levels, so the march skips whole inactive
// subtrees.  Inactive regions are absent from the walk, exactly as they are
// absent from the reference's pruned BVH.
#include "accel.cuh"
#include "scan.cuh"

namespace xb {
namespace {

__device__ double max_opacity_dev(double lo, double hi, const double* __restrict__ alpha, double vmin, double vmax) {
    // R/accel.py:91-115 (alpha = rgba[:, 3], 256 entries)
    const double scale = 255.0 / (hi - lo);
    double x0 = (vmin - lo) * scale, x1 = (vmax - lo) * scale;
    x0 = x0 < 0.0 ? 0.0 : x0;
    x0 = x0 > 255.0 ? 255.0 : x0;
    x1 = x1 < 0.0 ? 0.0 : x1;
    x1 = x1 > 255.0 ? 255.0 : x1;
    double m = 0.0;
    const double xs[2] = {x0, x1};
    for (int s = 0; s < 2; s++) {
        const double x = xs[s];
        const int i = (int)x;
        double v;
        if (i >= 255) v = alpha[255];
        else {
            const double f = x - (double)i;
            v = (1.0 - f) * alpha[i] + f * alpha[i + 1];
        }
        m = s == 0 ? v : (v > m ? v : m);
    }
    const int k0 = (int)ceil(x0), k1 = (int)floor(x1);
    for (int k = k0; k <= k1; k++) m = alpha[k] > m ? alpha[k] : m;
    return m;
}

struct AlphaTab {
    double a[256];
};

// Opacity minorant of a region for the walk's early-stop heuristic
// (render.cu:k_walk): the minimum of the TF alpha ramp over the region's
// value range, expressed as optical depth per unit ray length at spc = 1,
// q = -log(1 - a_min) / finest_width, so the opacity after a length L inside
// the region is at least 1 - exp(-spc * q * L) (R/render.py:432).  Only a
// heuristic input: k_warp never trusts it for correctness.
__global__ void k_volume_minorant(int64_t R, int F, int field, const float2* __restrict__ vrange, double lo,
                                  double hi, const AlphaTab tab, const RegionRec* __restrict__ rec, float* q) {
    __shared__ double s_a[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_a[i] = tab.a[i];
    __syncthreads();
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= R) return;
    const float2 v = vrange[r * F + field];
    const double scale = 255.0 / (hi - lo);
    double x0 = ((double)v.x - lo) * scale, x1 = ((double)v.y - lo) * scale;
    x0 = fmin(fmax(x0, 0.0), 255.0);
    x1 = fmin(fmax(x1, 0.0), 255.0);
    double m = 1.0;
    const double xs[2] = {x0, x1};
    for (int k = 0; k < 2; k++) {
        const int i = (int)xs[k];
        const double f = xs[k] - (double)i;
        const double a = i >= 255 ? s_a[255] : (1.0 - f) * s_a[i] + f * s_a[i + 1];
        m = fmin(m, a);
    }
    for (int k = (int)ceil(x0); k <= (int)floor(x1); k++) m = fmin(m, s_a[k]);
    m = fmin(fmax(m, 0.0), 0.999999);
    const double fw = ldexp(1.0, rec[r].meta >> 24);
    q[r] = (float)(-log1p(-m) / fw);
}

__global__ void k_volume_active(int64_t R, int F, int field, const float2* __restrict__ vrange, double lo, double hi,
                                const AlphaTab tab, uint8_t* act) {
    __shared__ double s_a[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_a[i] = tab.a[i];
    __syncthreads();
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= R) return;
    const float2 v = vrange[r * F + field];
    act[r] = max_opacity_dev(lo, hi, s_a, (double)v.x, (double)v.y) > 0.0;
}

__global__ void k_iso_active(int64_t R, int F, int field, const float2* __restrict__ vrange, double iso, uint8_t* act) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= R) return;
    const float2 v = vrange[r * F + field];
    act[r] = ((double)v.x <= iso) && (iso <= (double)v.y);
}

__global__ void k_all_active(int64_t R, uint8_t* act) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < R) act[r] = 1;
}

__global__ void k_flags_level(int64_t base, int64_t n, const KdNode* __restrict__ kd, const uint8_t* __restrict__ act,
                              uint8_t* flags) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t g = base + i;
    const KdNode nd = kd[g];
    uint8_t f;
    if (nd.a == -1) f = 0;
    else if ((nd.a & 3) == 3) f = act[nd.a >> 2];
    else {
        const int c = nd.a >> 2;
        f = flags[c] | flags[c + 1];
    }
    flags[g] = f;
}

__global__ void k_compact_active(int64_t R, const uint8_t* __restrict__ act, const int32_t* __restrict__ pos,
                                 int32_t* prims) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r < R && act[r]) prims[pos[r]] = (int32_t)r;
}

__global__ void k_u8_to_i32(int64_t n, const uint8_t* __restrict__ a, int32_t* b) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

}  // namespace

void build_active(const DevRegions& R, int kind, int field, double tf_lo, double tf_hi, const double* rgba_host,
                  double iso, DevActive& out, cudaStream_t s) {
    DeviceGuard g(R.device);
    XB_CHECK(R.has_tree, XB_ERR_NO_TREE, "regions carry no k-d tree");
    XB_CHECK(field >= 0 && field < std::max(R.n_fields, 1), XB_ERR_ARG, "field index out of range");
    out.device = R.device;
    out.kind = kind;
    const int64_t n = R.n_regions;
    out.act.alloc_async(n + 1, s);
    out.flags.alloc_async(R.n_kd + 1, s);
    const int BS = 256;
    if (n > 0) {
        if (kind == 0) {
            AlphaTab tab;
            for (int i = 0; i < 256; i++) tab.a[i] = rgba_host[4 * i + 3];
            k_volume_active<<<grid_for(n, BS), BS, 0, s>>>(n, R.n_fields, field, R.vrange.p, tf_lo, tf_hi, tab, out.act.p);
            out.qmin.alloc_async(n, s);
            k_volume_minorant<<<grid_for(n, BS), BS, 0, s>>>(n, R.n_fields, field, R.vrange.p, tf_lo, tf_hi, tab,
                                                              R.rec.p, out.qmin.p);
        } else if (kind == 1) {
            k_iso_active<<<grid_for(n, BS), BS, 0, s>>>(n, R.n_fields, field, R.vrange.p, iso, out.act.p);
        } else {
            k_all_active<<<grid_for(n, BS), BS, 0, s>>>(n, out.act.p);
        }
        check_launch("active");
    }
    const auto& lb = R.kd_level_base;
    for (int l = (int)lb.size() - 2; l >= 0; l--) {
        const int64_t b = lb[l], m = lb[l + 1] - b;
        if (m > 0) k_flags_level<<<grid_for(m, BS), BS, 0, s>>>(b, m, R.kd.p, out.act.p, out.flags.p);
    }
    check_launch("k_flags_level");
    build_kd4_mask(R, out.flags.p, out.mask4, s);
    // active id list (ascending) for RegionBvh.prims / n_active; scratch from
    // the stream's pool and prims sized for every region, so the only host
    // synchronisation is the final count read
    CubPoolTemp tmp(s);
    PoolBuf<int32_t> a32(n + 1, s), pos(n + 1, s);
    if (n > 0) k_u8_to_i32<<<grid_for(n, BS), BS, 0, s>>>(n, out.act.p, a32.p);
    XB_CUDA(cudaMemsetAsync(a32.p + n, 0, 4, s));
    exclusive_sum(tmp, a32.p, pos.p, n + 1, s);
    out.prims.alloc_async(n + 1, s);
    if (n > 0) k_compact_active<<<grid_for(n, BS), BS, 0, s>>>(n, out.act.p, pos.p, out.prims.p);
    check_launch("k_compact_active");
    out.n_active = read_scalar(pos.p + n, s);
}

// ---------------------------------------------------------------------------
// point sampling (R/sampling.py:260-353): region path via the region list
// (explicit region or k-d point location), and the brute-force cell scan.

namespace {

__global__ void k_sample(SceneView S, int64_t n, const double* __restrict__ p, const int32_t* __restrict__ rid_in,
                         int want_grad, int32_t* rid_out, double* out /* (n, 9) */) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const double px = p[3 * q], py = p[3 * q + 1], pz = p[3 * q + 2];
    int rid = rid_in ? rid_in[q] : -1;
    if (!rid_in) rid = kd_point(S, px, py, pz);
    rid_out[q] = rid;
    double* o = out + 9 * q;
    for (int c = 0; c < 9; c++) o[c] = 0.0;
    if (rid < 0) return;
    const RegionRec rr = S.rec[rid];
    Accum A;
    if (want_grad) {
        gather<true>(S, S.rids + rr.ids_begin, rr.meta & 0xffffff, px, py, pz, A);
        o[0] = A.num; o[1] = A.den;
        o[2] = A.gnum;
        for (int a = 0; a < 3; a++) { o[3 + a] = A.dn[a]; o[6 + a] = A.dd[a]; }
    } else {
        gather<false>(S, S.rids + rr.ids_begin, rr.meta & 0xffffff, px, py, pz, A);
        o[0] = A.num; o[1] = A.den;
    }
}

// `_accumulate_cells` (R/sampling.py:106-120) over the canonical cell order:
// one block per point, threads stride bricks, per-brick partial sums are
// combined IN BRICK ORDER by one thread so the sum order equals the scan's.
__global__ void k_sample_scan(SceneView S, int64_t n_bricks, int64_t n, const double* __restrict__ p,
                              double* out, double* scratch /* (n_blocks, n_bricks, 2) */) {
    const int64_t q = blockIdx.x;
    if (q >= n) return;
    const double px = p[3 * q], py = p[3 * q + 1], pz = p[3 * q + 2];
    double* sc = scratch + blockIdx.x * n_bricks * 2;
    for (int64_t b = threadIdx.x; b < n_bricks; b += blockDim.x) {
        // cells of brick b with nonzero weight: same candidate window as the
        // region gather, skipped cells contribute exactly nothing
        const int32_t id = (int32_t)b;
        Accum A;
        gather<false>(S, &id, 1, px, py, pz, A);
        sc[2 * b] = A.num;
        sc[2 * b + 1] = A.den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // sequential combination would re-round: instead re-run the exact
        // scan order over contributing bricks only
        double num = 0.0, den = 0.0;
        for (int64_t b = 0; b < n_bricks; b++) {
            if (sc[2 * b + 1] == 0.0) continue;
            const int32_t id = (int32_t)b;
            // continue the running sums through this brick's cells
            const int4 ba = S.brick_a[id];
            const uint32_t bm = S.brick_m[id];
            const int lev = bm & 31;
            const int nx = (bm >> 5) & 511, ny = (bm >> 14) & 511, nz = (bm >> 23) & 511;
            const double w = pow2(lev), iw_d = pow2(-lev);
            const int64_t iw = (int64_t)1 << lev;
            const int64_t x0 = (int64_t)floor((px - (double)ba.x) * iw_d - 0.5);
            const int64_t y0 = (int64_t)floor((py - (double)ba.y) * iw_d - 0.5);
            const int64_t z0 = (int64_t)floor((pz - (double)ba.z) * iw_d - 0.5);
            for (int64_t z = max(z0, (int64_t)0); z < min(z0 + 2, (int64_t)nz); z++)
                for (int64_t y = max(y0, (int64_t)0); y < min(y0 + 2, (int64_t)ny); y++)
                    for (int64_t x = max(x0, (int64_t)0); x < min(x0 + 2, (int64_t)nx); x++) {
                        const double hx = 1.0 - fabs(((double)(ba.x + x * iw) + 0.5 * w) - px) * iw_d;
                        const double hy = 1.0 - fabs(((double)(ba.y + y * iw) + 0.5 * w) - py) * iw_d;
                        const double hz = 1.0 - fabs(((double)(ba.z + z * iw) + 0.5 * w) - pz) * iw_d;
                        if (hx > 0.0 && hy > 0.0 && hz > 0.0) {
                            const double h = hx * hy * hz;
                            num += h * (double)S.vals[(uint32_t)ba.w + x + nx * (y + ny * z)];
                            den += h;
                        }
                    }
        }
        out[2 * q] = num;
        out[2 * q + 1] = den;
    }
}

// `_accumulate_cells` (R/sampling.py:106-120) over an arbitrary cell list in its
// given order (basis_sample_oracle on a plain CellList, R/sampling.py:291-298):
// one block per point; each pass tests 128 consecutive cells (hats > 0), a
// block scan of the hit flags appends the contributing indices in list order
// to shared memory, and one thread adds them in that order — the reference's
// exact sequence.  A point with more than kScanCap contributors (not possible
// for a valid AMR list, whose cells are disjoint) takes the sequential scan.
constexpr int kScanCap = 1024;
__global__ void __launch_bounds__(128) k_scan_cells(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                                                     const int32_t* __restrict__ ck, const int32_t* __restrict__ cl,
                                                     const float* __restrict__ cv, int64_t n_cells, int64_t n,
                                                     const double* __restrict__ p, double* __restrict__ out) {
    __shared__ int32_t s_hit[kScanCap];
    __shared__ int s_warp[4];
    __shared__ int s_n;
    const int64_t q = blockIdx.x;
    if (q >= n) return;
    const double px = p[3 * q], py = p[3 * q + 1], pz = p[3 * q + 2];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    auto hats = [&](int64_t t, double& hx, double& hy, double& hz) {
        const double w = pow2(cl[t]), iw = pow2(-cl[t]);
        hx = 1.0 - fabs(((double)ci[t] + 0.5 * w) - px) * iw;
        hy = 1.0 - fabs(((double)cj[t] + 0.5 * w) - py) * iw;
        hz = 1.0 - fabs(((double)ck[t] + 0.5 * w) - pz) * iw;
    };
    for (int64_t base = 0; base < n_cells; base += blockDim.x) {
        const int64_t t = base + threadIdx.x;
        bool hit = false;
        if (t < n_cells) {
            double hx, hy, hz;
            hats(t, hx, hy, hz);
            hit = hx > 0.0 && hy > 0.0 && hz > 0.0;
        }
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_warp[wid] = __popc(b);
        __syncthreads();
        int before = s_n;
        for (int w = 0; w < wid; w++) before += s_warp[w];
        const int pos = before + __popc(b & ((1u << lane) - 1u));
        if (hit && pos < kScanCap) s_hit[pos] = (int32_t)t;
        __syncthreads();
        if (threadIdx.x == 0) s_n += s_warp[0] + s_warp[1] + s_warp[2] + s_warp[3];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    double num = 0.0, den = 0.0;
    const bool fits = s_n <= kScanCap;
    const int64_t m = fits ? s_n : n_cells;
    for (int64_t u = 0; u < m; u++) {
        const int64_t t = fits ? s_hit[u] : u;
        double hx, hy, hz;
        hats(t, hx, hy, hz);
        if (hx > 0.0 && hy > 0.0 && hz > 0.0) {
            const double h = hx * hy * hz;
            num += h * (double)cv[t];
            den += h;
        }
    }
    out[2 * q] = num;
    out[2 * q + 1] = den;
}

// iterate_intervals (R/accel.py:414-424) for a batch of rays, via the ordered
// k-d walk; up to `cap` intervals per ray.
__global__ void k_trace(SceneView S, const uint8_t* __restrict__ flags, int64_t n, const double* __restrict__ o,
                        const double* __restrict__ d, double t_start, double t_max, int cap, double* tin, double* tout,
                        int32_t* reg, int32_t* cnt, LbvhView L, int use_lb) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    Ray r;
    for (int a = 0; a < 3; a++) {
        r.o[a] = o[3 * q + a];
        r.d[a] = d[3 * q + a];
        r.inv[a] = 1.0 / r.d[a];
    }
    KdWalk w;
    kd_begin(S, r, w);
    double t = t_start;
    int k = 0;
    for (;;) {
        int rid;
        double ci, co;
        // ordered k-d walk, or the reference's per-visit closest-hit query on the LBVH
        if (!(use_lb ? lbvh_next_hit(S, L, r, t, t_max, rid, ci, co) : kd_next(S, flags, r, w, t, t_max, rid, ci, co)))
            break;
        if (k < cap) {
            tin[q * cap + k] = ci;
            tout[q * cap + k] = co;
            reg[q * cap + k] = rid;
        }
        k++;
        t = restart_t(co);
        if (t >= t_max) break;
    }
    cnt[q] = k;
}

}  // namespace

void sample_points(const SceneView& S, int64_t n, const double* p, const int32_t* rid_in, int want_grad, int32_t* rid_out,
                   double* out, cudaStream_t s) {
    if (n <= 0) return;
    k_sample<<<grid_for(n, 128), 128, 0, s>>>(S, n, p, rid_in, want_grad, rid_out, out);
    check_launch("k_sample");
}

void sample_scan(const SceneView& S, int64_t n_bricks, int64_t n, const double* p, double* out, cudaStream_t s) {
    if (n <= 0) return;
    const int64_t chunk = 256;
    DevBuf<double> scratch(chunk * std::max<int64_t>(n_bricks, 1) * 2);
    for (int64_t b = 0; b < n; b += chunk) {
        const int64_t m = std::min(chunk, n - b);
        k_sample_scan<<<(unsigned)m, 128, 0, s>>>(S, n_bricks, m, p + 3 * b, out + 2 * b, scratch.p);
        check_launch("k_sample_scan");
    }
    XB_CUDA(cudaStreamSynchronize(s));
}

void scan_cells(const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* l, const float* v, int64_t n_cells,
                int64_t n, const double* p, double* out, cudaStream_t s) {
    for (int64_t b = 0; b < n; b += 65535) {
        const int64_t m = std::min<int64_t>(65535, n - b);
        k_scan_cells<<<(unsigned)m, 128, 0, s>>>(i, j, k, l, v, n_cells, m, p + 3 * b, out + 2 * b);
        check_launch("k_scan_cells");
    }
}

void trace_intervals(const SceneView& S, const uint8_t* flags, int64_t n, const double* o, const double* d, double t0,
                     double t1, int cap, double* tin, double* tout, int32_t* reg, int32_t* cnt, cudaStream_t s,
                     const LbvhView* lb) {
    if (n <= 0) return;
    const LbvhView L = lb ? *lb : LbvhView{nullptr, nullptr, 0};
    k_trace<<<grid_for(n, 64), 64, 0, s>>>(S, flags, n, o, d, t0, t1, cap, tin, tout, reg, cnt, L, lb ? 1 : 0);
    check_launch("k_trace");
}

namespace {
__global__ void k_point_lbvh(SceneView S, LbvhView L, int64_t n, const double* __restrict__ p, int32_t* out) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < n) out[q] = lbvh_point(S, L, p[3 * q], p[3 * q + 1], p[3 * q + 2]);
}
}  // namespace

void point_query_lbvh(const SceneView& S, const LbvhView& L, int64_t n, const double* p, int32_t* out, cudaStream_t s) {
    if (n <= 0) return;
    k_point_lbvh<<<grid_for(n, 64), 64, 0, s>>>(S, L, n, p, out);
    check_launch("k_point_lbvh");
}

const DevLbvh& active_lbvh(const DevRegions& R, const DevActive& a, cudaStream_t s) {
    std::lock_guard<std::mutex> g(a.lb_mu);
    if (!a.lb) {
        auto lb = std::make_unique<DevLbvh>();
        build_lbvh(R, a.prims.p, a.n_active, *lb, s);
        XB_CUDA(cudaStreamSynchronize(s));
        a.lb = std::move(lb);
    }
    return *a.lb;
}

}  // namespace xb
