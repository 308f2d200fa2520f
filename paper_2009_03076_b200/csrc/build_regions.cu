// build_regions.cu — GPU Active-Brick-Region builder (paper §3.2).
//
// Restates `build_regions` + `_region_metadata` (R/regions.py:82-213,
// R/ = /root/reference/pkg/src/amrvol/) bit-exactly, but level-synchronously:
// every frontier node of one tree level is processed by the same kernels, all
// fragments (clipped brick supports, half-unit ints) of the level live in one
// SoA array grouped by node.  The reference's DFS (right pushed first, so the
// left child is finished first) numbers regions in left-first preorder of the
// non-empty leaves; we recover that order after the build by a bottom-up
// count / top-down offset pass over the recorded tree (in-order renumbering).
//
// Per node (R/regions.py:116-149):
//   axes by descending width (stable), first axis that has a candidate face
//   strictly inside the node; plane = candidate minimising |2f-(lo+hi)|, ties
//   to the lower f; left gets fragments with flo < plane (hi clipped), right
//   gets fhi > plane (lo clipped); no candidate -> leaf (dropped if empty).
// Fragment order inside a node never changes (stable scatter), so each
// leaf's brick-id list is already ascending (the reference's np.sort).
#include "common.cuh"
#include "scan.cuh"
#include "accel.cuh"
#include <algorithm>
#include <cstdlib>

namespace xb {
namespace {

constexpr uint64_t kNoKey = ~0ull;
constexpr int32_t kHalfMax = 1 << 29;  // |half-unit coordinate| bound for packed keys

struct Frags {
    DevBuf<int32_t> lo[3], hi[3], id, node;
    void ensure(size_t n) {
        for (int a = 0; a < 3; a++) { lo[a].ensure(n); hi[a].ensure(n); }
        id.ensure(n);
        node.ensure(n);
    }
};

struct Nodes {
    DevBuf<int32_t> lo[3], hi[3], fs, fc;  // box, fragment start / count
    void ensure(size_t n) {
        for (int a = 0; a < 3; a++) { lo[a].ensure(n); hi[a].ensure(n); }
        fs.ensure(n);
        fc.ensure(n);
    }
};

__global__ void k_init_supports(int64_t B, const int32_t* __restrict__ lower, const int32_t* __restrict__ level,
                                const int32_t* __restrict__ dims, int32_t* lo0, int32_t* lo1, int32_t* lo2, int32_t* hi0,
                                int32_t* hi1, int32_t* hi2, int32_t* id, int32_t* node) {
    // _support_boxes_halfunits, R/regions.py:82-87
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    int64_t w = (int64_t)1 << level[b];
    int32_t* los[3] = {lo0, lo1, lo2};
    int32_t* his[3] = {hi0, hi1, hi2};
    for (int a = 0; a < 3; a++) {
        int64_t l = lower[3 * b + a], h = l + (int64_t)dims[3 * b + a] * w;
        los[a][b] = (int32_t)(2 * l - w);
        his[a][b] = (int32_t)(2 * h + w);
    }
    id[b] = (int32_t)b;
    node[b] = 0;
}

__device__ __forceinline__ uint64_t face_key(int32_t f, int32_t lo, int32_t hi) {
    int64_t d = 2 * (int64_t)f - ((int64_t)lo + hi);
    if (d < 0) d = -d;
    return ((uint64_t)d << 32) | (uint32_t)(f + kHalfMax);
}

// candidate faces: per node and axis, min over (|2f-(lo+hi)|, f)
__global__ void k_candidates(int64_t F, const int32_t* __restrict__ flo0, const int32_t* __restrict__ flo1,
                             const int32_t* __restrict__ flo2, const int32_t* __restrict__ fhi0,
                             const int32_t* __restrict__ fhi1, const int32_t* __restrict__ fhi2,
                             const int32_t* __restrict__ fnode, const int32_t* __restrict__ nlo0,
                             const int32_t* __restrict__ nlo1, const int32_t* __restrict__ nlo2,
                             const int32_t* __restrict__ nhi0, const int32_t* __restrict__ nhi1,
                             const int32_t* __restrict__ nhi2, int64_t M, unsigned long long* keys) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool valid = t < F;
    int nd = valid ? fnode[t] : -1;
    uint64_t best[3] = {kNoKey, kNoKey, kNoKey};
    if (valid) {
        const int32_t* flo[3] = {flo0, flo1, flo2};
        const int32_t* fhi[3] = {fhi0, fhi1, fhi2};
        const int32_t* nlo[3] = {nlo0, nlo1, nlo2};
        const int32_t* nhi[3] = {nhi0, nhi1, nhi2};
#pragma unroll
        for (int a = 0; a < 3; a++) {
            int32_t lo = nlo[a][nd], hi = nhi[a][nd];
            int32_t f0 = flo[a][t], f1 = fhi[a][t];
            if (f0 > lo && f0 < hi) best[a] = min(best[a], face_key(f0, lo, hi));
            if (f1 > lo && f1 < hi) best[a] = min(best[a], face_key(f1, lo, hi));
        }
    }
    const unsigned full = 0xffffffffu;
    bool uni = warp_uniform(full, nd);
    if (uni) {
#pragma unroll
        for (int a = 0; a < 3; a++)
            for (int o = 16; o > 0; o >>= 1) best[a] = min(best[a], (uint64_t)__shfl_xor_sync(full, (unsigned long long)best[a], o));
        if ((threadIdx.x & 31) == 0 && nd >= 0)
            for (int a = 0; a < 3; a++)
                if (best[a] != kNoKey) atomicMin(&keys[a * M + nd], (unsigned long long)best[a]);
    } else if (valid) {
        for (int a = 0; a < 3; a++)
            if (best[a] != kNoKey) atomicMin(&keys[a * M + nd], (unsigned long long)best[a]);
    }
}

// per node: choose axis/plane or leaf
__global__ void k_decide(int64_t M, const unsigned long long* __restrict__ keys, const int32_t* __restrict__ nlo0,
                         const int32_t* __restrict__ nlo1, const int32_t* __restrict__ nlo2,
                         const int32_t* __restrict__ nhi0, const int32_t* __restrict__ nhi1,
                         const int32_t* __restrict__ nhi2, const int32_t* __restrict__ fc, int32_t* n_axis,
                         int32_t* n_plane, int32_t* n_split /* M+1 */, int32_t* n_leafc /* M+1 */) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t w[3] = {(int64_t)nhi0[i] - nlo0[i], (int64_t)nhi1[i] - nlo1[i], (int64_t)nhi2[i] - nlo2[i]};
    int ord[3] = {0, 1, 2};  // np.argsort(-(rhi - rlo), kind="stable")
    for (int x = 1; x < 3; x++)
        for (int y = x; y > 0 && w[ord[y]] > w[ord[y - 1]]; y--) { int tt = ord[y]; ord[y] = ord[y - 1]; ord[y - 1] = tt; }
    int axis = -1;
    int32_t plane = 0;
    for (int o = 0; o < 3; o++) {
        uint64_t k = keys[ord[o] * M + i];
        if (k != kNoKey) {
            axis = ord[o];
            plane = (int32_t)((uint32_t)(k & 0xffffffffu)) - kHalfMax;
            break;
        }
    }
    n_axis[i] = axis;
    n_plane[i] = plane;
    n_split[i] = axis >= 0 ? 1 : 0;
    n_leafc[i] = axis >= 0 ? 0 : fc[i];
}

__global__ void k_flags(int64_t F, const int32_t* __restrict__ fnode, const int32_t* __restrict__ n_axis,
                        const int32_t* __restrict__ n_plane, const int32_t* __restrict__ flo0,
                        const int32_t* __restrict__ flo1, const int32_t* __restrict__ flo2,
                        const int32_t* __restrict__ fhi0, const int32_t* __restrict__ fhi1,
                        const int32_t* __restrict__ fhi2, int32_t* gl, int32_t* gr) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= F) return;
    int nd = fnode[t];
    int a = n_axis[nd];
    int l = 0, r = 0;
    if (a >= 0) {
        int32_t p = n_plane[nd];
        int32_t lo = a == 0 ? flo0[t] : (a == 1 ? flo1[t] : flo2[t]);
        int32_t hi = a == 0 ? fhi0[t] : (a == 1 ? fhi1[t] : fhi2[t]);
        l = lo < p;
        r = hi > p;
    }
    gl[t] = l;
    gr[t] = r;
}

// per node: child fragment counts (for scan) from the flag scans
__global__ void k_child_counts(int64_t M, const int32_t* __restrict__ fs, const int32_t* __restrict__ fc,
                               const int32_t* __restrict__ n_split, const int32_t* __restrict__ sl,
                               const int32_t* __restrict__ sr, int32_t* nl, int32_t* cnt /* M+1 */) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int32_t b = fs[i], e = fs[i] + fc[i];
    int32_t l = sl[e] - sl[b], r = sr[e] - sr[b];
    nl[i] = l;
    cnt[i] = n_split[i] ? l + r : 0;
}

__global__ void k_scatter(int64_t F, const int32_t* __restrict__ fnode, const int32_t* __restrict__ n_axis,
                          const int32_t* __restrict__ n_plane, const int32_t* __restrict__ fs,
                          const int32_t* __restrict__ nl, const int32_t* __restrict__ child_start,
                          const int32_t* __restrict__ split_rank, const int32_t* __restrict__ leaf_off,
                          const int32_t* __restrict__ sl, const int32_t* __restrict__ sr, const int32_t* flo0,
                          const int32_t* flo1, const int32_t* flo2, const int32_t* fhi0, const int32_t* fhi1,
                          const int32_t* fhi2, const int32_t* fid, int32_t* olo0, int32_t* olo1, int32_t* olo2,
                          int32_t* ohi0, int32_t* ohi1, int32_t* ohi2, int32_t* oid, int32_t* onode,
                          int32_t* leaf_store, int64_t leaf_base) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= F) return;
    int nd = fnode[t];
    int a = n_axis[nd];
    int32_t lo[3] = {flo0[t], flo1[t], flo2[t]};
    int32_t hi[3] = {fhi0[t], fhi1[t], fhi2[t]};
    int32_t id = fid[t];
    if (a < 0) {  // leaf: keep the brick id, in order
        leaf_store[leaf_base + leaf_off[nd] + (t - fs[nd])] = id;
        return;
    }
    int32_t p = n_plane[nd];
    int32_t b = fs[nd];
    int32_t child = 2 * split_rank[nd];
    if (lo[a] < p) {
        int64_t d = child_start[nd] + (sl[t] - sl[b]);
        int32_t h = hi[a] < p ? hi[a] : p;  // np.minimum(lhi, plane)
        olo0[d] = lo[0]; olo1[d] = lo[1]; olo2[d] = lo[2];
        ohi0[d] = a == 0 ? h : hi[0]; ohi1[d] = a == 1 ? h : hi[1]; ohi2[d] = a == 2 ? h : hi[2];
        oid[d] = id;
        onode[d] = child;
    }
    if (hi[a] > p) {
        int64_t d = child_start[nd] + nl[nd] + (sr[t] - sr[b]);
        int32_t l = lo[a] > p ? lo[a] : p;  // np.maximum(rlo, plane)
        olo0[d] = a == 0 ? l : lo[0]; olo1[d] = a == 1 ? l : lo[1]; olo2[d] = a == 2 ? l : lo[2];
        ohi0[d] = hi[0]; ohi1[d] = hi[1]; ohi2[d] = hi[2];
        oid[d] = id;
        onode[d] = child + 1;
    }
}

// tree record of this level + child node boxes/ranges for the next level
struct TreeRec {
    DevBuf<int32_t> kind;        // 0 split, 1 leaf with bricks, 2 cavity
    DevBuf<int32_t> child;       // tree index of left child (split)
    DevBuf<int32_t> axis, plane;
    DevBuf<int32_t> lo, hi;      // (T,3) boxes (leaves need them; kept for all)
    DevBuf<int32_t> leaf_first, leaf_count;
    DevBuf<int64_t> cnt_reg, cnt_ids, off_reg, off_ids;
};

__global__ void k_record(int64_t M, int64_t base, int64_t next_base, const int32_t* __restrict__ n_axis,
                         const int32_t* __restrict__ n_plane, const int32_t* __restrict__ split_rank,
                         const int32_t* __restrict__ fc, const int32_t* __restrict__ leaf_off, int64_t leaf_base,
                         const int32_t* nlo0, const int32_t* nlo1, const int32_t* nlo2, const int32_t* nhi0,
                         const int32_t* nhi1, const int32_t* nhi2, const int32_t* __restrict__ child_start,
                         const int32_t* __restrict__ nl, const int32_t* __restrict__ cnt, int32_t* kind, int32_t* child,
                         int32_t* axis, int32_t* plane, int32_t* tlo, int32_t* thi, int32_t* leaf_first,
                         int32_t* leaf_count, int32_t* clo0, int32_t* clo1, int32_t* clo2, int32_t* chi0, int32_t* chi1,
                         int32_t* chi2, int32_t* cfs, int32_t* cfc) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t g = base + i;
    int a = n_axis[i];
    int32_t lo[3] = {nlo0[i], nlo1[i], nlo2[i]};
    int32_t hi[3] = {nhi0[i], nhi1[i], nhi2[i]};
    for (int c = 0; c < 3; c++) { tlo[3 * g + c] = lo[c]; thi[3 * g + c] = hi[c]; }
    axis[g] = a;
    plane[g] = n_plane[i];
    if (a < 0) {
        kind[g] = fc[i] > 0 ? 1 : 2;
        child[g] = -1;
        leaf_first[g] = (int32_t)(leaf_base + leaf_off[i]);
        leaf_count[g] = fc[i];
        return;
    }
    kind[g] = 0;
    int32_t c = 2 * split_rank[i];
    child[g] = (int32_t)(next_base + c);
    leaf_first[g] = 0;
    leaf_count[g] = 0;
    int32_t p = n_plane[i];
    // left child box: hi[axis] = plane ; right: lo[axis] = plane (not tightened, R/regions.py:143-146)
    int32_t* clo[3] = {clo0, clo1, clo2};
    int32_t* chi[3] = {chi0, chi1, chi2};
    for (int x = 0; x < 3; x++) {
        clo[x][c] = lo[x]; chi[x][c] = hi[x];
        clo[x][c + 1] = lo[x]; chi[x][c + 1] = hi[x];
    }
    chi[a][c] = p;
    clo[a][c + 1] = p;
    cfs[c] = child_start[i];
    cfc[c] = nl[i];
    cfs[c + 1] = child_start[i] + nl[i];
    cfc[c + 1] = cnt[i] - nl[i];
}

__global__ void k_bottom_up(int64_t base, int64_t M, const int32_t* __restrict__ kind, const int32_t* __restrict__ child,
                            const int32_t* __restrict__ leaf_count, int64_t* cnt_reg, int64_t* cnt_ids) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t g = base + i;
    if (kind[g] == 0) {
        int c = child[g];
        cnt_reg[g] = cnt_reg[c] + cnt_reg[c + 1];
        cnt_ids[g] = cnt_ids[c] + cnt_ids[c + 1];
    } else {
        cnt_reg[g] = kind[g] == 1 ? 1 : 0;
        cnt_ids[g] = kind[g] == 1 ? leaf_count[g] : 0;
    }
}

__global__ void k_top_down(int64_t base, int64_t M, const int32_t* __restrict__ kind, const int32_t* __restrict__ child,
                           const int64_t* __restrict__ cnt_reg, const int64_t* __restrict__ cnt_ids, int64_t* off_reg,
                           int64_t* off_ids) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t g = base + i;
    if (kind[g] != 0) return;
    int c = child[g];
    off_reg[c] = off_reg[g];
    off_ids[c] = off_ids[g];
    off_reg[c + 1] = off_reg[g] + cnt_reg[c];
    off_ids[c + 1] = off_ids[g] + cnt_ids[c];
}

__global__ void k_finalize(int64_t T, const int32_t* __restrict__ kind, const int32_t* __restrict__ child,
                           const int32_t* __restrict__ axis, const int32_t* __restrict__ plane,
                           const int32_t* __restrict__ tlo, const int32_t* __restrict__ thi,
                           const int32_t* __restrict__ leaf_first, const int32_t* __restrict__ leaf_count,
                           const int64_t* __restrict__ off_reg, const int64_t* __restrict__ off_ids,
                           const int32_t* __restrict__ leaf_store, const int32_t* __restrict__ blevel, KdNode* kd,
                           RegionRec* rec, int32_t* ids, double* lo, double* hi, int64_t* brick_off) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= T) return;
    KdNode nd;
    if (kind[g] == 0) {
        nd.a = (child[g] << 2) | axis[g];
        nd.b = plane[g];
    } else if (kind[g] == 2) {
        nd.a = -1;
        nd.b = 0;
    } else {
        int64_t r = off_reg[g];
        int64_t ib = off_ids[g];
        int32_t n = leaf_count[g];
        int minlev = 1 << 30;
        for (int32_t t = 0; t < n; t++) {
            int32_t b = leaf_store[leaf_first[g] + t];
            ids[ib + t] = b;
            minlev = min(minlev, blevel[b]);
        }
        RegionRec rr;
        for (int c = 0; c < 3; c++) {
            rr.lo[c] = tlo[3 * g + c];
            rr.hi[c] = thi[3 * g + c];
            lo[3 * r + c] = (double)tlo[3 * g + c] / 2.0;  // lo_h / 2.0, exact
            hi[3 * r + c] = (double)thi[3 * g + c] / 2.0;
        }
        rr.ids_begin = (int32_t)ib;
        rr.meta = n | (minlev << 24);
        rec[r] = rr;
        brick_off[r] = ib;
        nd.a = (int32_t)((r << 2) | 3);
        nd.b = 0;
    }
    kd[g] = nd;
}

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    return (q * b != a && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// _region_metadata (R/regions.py:174-213): one warp per region, lanes stride
// over every (brick, cell) whose support overlaps the region interior.
__global__ void k_metadata(int64_t R, int F, const RegionRec* __restrict__ rec, const int32_t* __restrict__ ids,
                           const int32_t* __restrict__ blower, const int32_t* __restrict__ blevel,
                           const int32_t* __restrict__ bdims, const int64_t* __restrict__ boff,
                           const float* __restrict__ vals, int64_t N, float2* vrange, double* vr64, double* finest) {
    int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= R) return;
    RegionRec rr = rec[warp];
    int nids = rr.meta & 0xffffff;
    constexpr int FMAX = 8;
    float mn[FMAX], mx[FMAX];
    for (int f = 0; f < FMAX; f++) { mn[f] = INFINITY; mx[f] = -INFINITY; }
    for (int t = 0; t < nids; t++) {
        int b = ids[rr.ids_begin + t];
        int lev = blevel[b];
        int64_t w_h = (int64_t)2 << lev, half_h = (int64_t)1 << lev;
        int64_t i0[3], i1[3], n3[3];
        for (int a = 0; a < 3; a++) {
            n3[a] = bdims[3 * b + a];
            int64_t blh = 2 * (int64_t)blower[3 * b + a];
            int64_t x0 = floordiv((int64_t)rr.lo[a] - blh - half_h, w_h);
            int64_t x1 = floordiv((int64_t)rr.hi[a] - blh + half_h - 1, w_h);
            i0[a] = x0 > 0 ? x0 : 0;
            i1[a] = x1 < n3[a] - 1 ? x1 : n3[a] - 1;
        }
        int64_t ex = i1[0] - i0[0] + 1, ey = i1[1] - i0[1] + 1, ez = i1[2] - i0[2] + 1;
        if (ex <= 0 || ey <= 0 || ez <= 0) continue;
        int64_t total = ex * ey * ez;
        int64_t base = boff[b];
        for (int64_t q = lane; q < total; q += 32) {
            int64_t x = i0[0] + q % ex, y = i0[1] + (q / ex) % ey, z = i0[2] + q / (ex * ey);
            int64_t slot = base + x + n3[0] * (y + n3[1] * z);
            for (int f = 0; f < F && f < FMAX; f++) {
                float v = vals[f * N + slot];
                mn[f] = fminf(mn[f], v);
                mx[f] = fmaxf(mx[f], v);
            }
        }
    }
    for (int f = 0; f < F && f < FMAX; f++) {
        for (int o = 16; o > 0; o >>= 1) {
            mn[f] = fminf(mn[f], __shfl_xor_sync(0xffffffffu, mn[f], o));
            mx[f] = fmaxf(mx[f], __shfl_xor_sync(0xffffffffu, mx[f], o));
        }
        if (lane == 0) {
            vrange[warp * F + f] = make_float2(mn[f], mx[f]);
            vr64[(warp * F + f) * 2] = (double)mn[f];
            vr64[(warp * F + f) * 2 + 1] = (double)mx[f];
        }
    }
    if (lane == 0) finest[warp] = ldexp(1.0, rr.meta >> 24);
}

}  // namespace

// Build regions + k-d tree for a device model.  Synchronous on `s`.
void build_regions_device(const DevModel& m, DevRegions& out, cudaStream_t s) {
    DeviceGuard g(m.device);
    out = DevRegions();
    out.device = m.device;
    out.n_fields = m.n_fields;
    XB_CHECK(m.n_fields <= 8, XB_ERR_RANGE, "build_regions: at most 8 fields supported on the GPU");
    const int64_t B = m.n_bricks;
    out.brick_off.alloc(1);
    if (B == 0) {
        XB_CUDA(cudaMemsetAsync(out.brick_off.p, 0, sizeof(int64_t), s));
        XB_CUDA(cudaStreamSynchronize(s));
        out.has_tree = true;  // empty tree: render sees no regions
        return;
    }
    {
        // half-unit supports must stay inside +-2^29 for the packed face keys
        int64_t amax = std::max<int64_t>(std::llabs((long long)m.coord_min), std::llabs((long long)m.coord_max));
        XB_CHECK(2 * amax + (1ll << m.max_level) < (int64_t)kHalfMax, XB_ERR_RANGE,
                 "build_regions: brick coordinates exceed the supported half-unit range (|x| < 2^28)");
    }
    CubTemp tmp;
    Frags fa, fb;
    Nodes na, nb;
    fa.ensure(B);
    na.ensure(1);
    const int BS = 256;
    k_init_supports<<<grid_for(B, BS), BS, 0, s>>>(B, m.lower.p, m.level.p, m.dims.p, fa.lo[0].p, fa.lo[1].p, fa.lo[2].p,
                                                    fa.hi[0].p, fa.hi[1].p, fa.hi[2].p, fa.id.p, fa.node.p);
    check_launch("k_init_supports");
    // root box = union of supports
    DevBuf<int32_t> red1;
    int32_t root_lo[3], root_hi[3];
    for (int a = 0; a < 3; a++) {
        root_lo[a] = reduce_min(tmp, fa.lo[a].p, B, red1, s);
        root_hi[a] = reduce_max(tmp, fa.hi[a].p, B, red1, s);
        XB_CUDA(cudaMemcpyAsync(na.lo[a].p, &root_lo[a], 4, cudaMemcpyHostToDevice, s));
        XB_CUDA(cudaMemcpyAsync(na.hi[a].p, &root_hi[a], 4, cudaMemcpyHostToDevice, s));
        out.root_lo[a] = root_lo[a];
        out.root_hi[a] = root_hi[a];
    }
    int32_t zero = 0, b32 = (int32_t)B;
    XB_CUDA(cudaMemcpyAsync(na.fs.p, &zero, 4, cudaMemcpyHostToDevice, s));
    XB_CUDA(cudaMemcpyAsync(na.fc.p, &b32, 4, cudaMemcpyHostToDevice, s));

    TreeRec tr;
    DevBuf<int32_t> leaf_store;
    int64_t T = 0, leaf_total = 0;
    int64_t M = 1, F = B;
    int depth = 0;
    DevBuf<unsigned long long> keys;
    DevBuf<int32_t> n_axis, n_plane, n_split, split_rank, n_leafc, leaf_off, nl, cnt, child_start, gl, gr, sl, sr;
    std::vector<int64_t> level_base;
    while (M > 0) {
        XB_CHECK(F < (1ll << 31) - 1, XB_ERR_RANGE, "build_regions: fragment count exceeds 2^31");
        level_base.push_back(T);
        depth++;
        keys.ensure(3 * M);
        XB_CUDA(cudaMemsetAsync(keys.p, 0xff, 3 * M * sizeof(unsigned long long), s));
        if (F > 0) k_candidates<<<grid_for(F, BS), BS, 0, s>>>(F, fa.lo[0].p, fa.lo[1].p, fa.lo[2].p, fa.hi[0].p, fa.hi[1].p,
                                                     fa.hi[2].p, fa.node.p, na.lo[0].p, na.lo[1].p, na.lo[2].p,
                                                     na.hi[0].p, na.hi[1].p, na.hi[2].p, M, keys.p);
        check_launch("k_candidates");
        n_axis.ensure(M); n_plane.ensure(M); n_split.ensure(M + 1); n_leafc.ensure(M + 1);
        split_rank.ensure(M + 1); leaf_off.ensure(M + 1); nl.ensure(M); cnt.ensure(M + 1); child_start.ensure(M + 1);
        k_decide<<<grid_for(M, BS), BS, 0, s>>>(M, keys.p, na.lo[0].p, na.lo[1].p, na.lo[2].p, na.hi[0].p, na.hi[1].p,
                                                na.hi[2].p, na.fc.p, n_axis.p, n_plane.p, n_split.p, n_leafc.p);
        check_launch("k_decide");
        XB_CUDA(cudaMemsetAsync(n_split.p + M, 0, 4, s));
        XB_CUDA(cudaMemsetAsync(n_leafc.p + M, 0, 4, s));
        exclusive_sum(tmp, n_split.p, split_rank.p, M + 1, s);
        exclusive_sum(tmp, n_leafc.p, leaf_off.p, M + 1, s);
        gl.ensure(F + 1); gr.ensure(F + 1); sl.ensure(F + 1); sr.ensure(F + 1);
        if (F > 0) k_flags<<<grid_for(F, BS), BS, 0, s>>>(F, fa.node.p, n_axis.p, n_plane.p, fa.lo[0].p, fa.lo[1].p, fa.lo[2].p,
                                               fa.hi[0].p, fa.hi[1].p, fa.hi[2].p, gl.p, gr.p);
        check_launch("k_flags");
        XB_CUDA(cudaMemsetAsync(gl.p + F, 0, 4, s));
        XB_CUDA(cudaMemsetAsync(gr.p + F, 0, 4, s));
        exclusive_sum(tmp, gl.p, sl.p, F + 1, s);
        exclusive_sum(tmp, gr.p, sr.p, F + 1, s);
        k_child_counts<<<grid_for(M, BS), BS, 0, s>>>(M, na.fs.p, na.fc.p, n_split.p, sl.p, sr.p, nl.p, cnt.p);
        check_launch("k_child_counts");
        XB_CUDA(cudaMemsetAsync(cnt.p + M, 0, 4, s));
        exclusive_sum(tmp, cnt.p, child_start.p, M + 1, s);
        int32_t n_splits = read_scalar(split_rank.p + M, s);
        int32_t leaf_frags = read_scalar(leaf_off.p + M, s);
        int32_t F_next = read_scalar(child_start.p + M, s);
        int64_t M_next = 2 * (int64_t)n_splits;
        // grow outputs
        grow_keep(leaf_store, leaf_total + leaf_frags, leaf_total, s);
        size_t Tn = T + M;
        grow_keep(tr.kind, Tn, T, s); grow_keep(tr.child, Tn, T, s); grow_keep(tr.axis, Tn, T, s);
        grow_keep(tr.plane, Tn, T, s); grow_keep(tr.lo, 3 * Tn, 3 * T, s); grow_keep(tr.hi, 3 * Tn, 3 * T, s);
        grow_keep(tr.leaf_first, Tn, T, s); grow_keep(tr.leaf_count, Tn, T, s);
        fb.ensure(F_next > 0 ? F_next : 1);
        nb.ensure(M_next > 0 ? M_next : 1);
        if (F > 0) k_scatter<<<grid_for(F, BS), BS, 0, s>>>(F, fa.node.p, n_axis.p, n_plane.p, na.fs.p, nl.p, child_start.p,
                                                 split_rank.p, leaf_off.p, sl.p, sr.p, fa.lo[0].p, fa.lo[1].p,
                                                 fa.lo[2].p, fa.hi[0].p, fa.hi[1].p, fa.hi[2].p, fa.id.p, fb.lo[0].p,
                                                 fb.lo[1].p, fb.lo[2].p, fb.hi[0].p, fb.hi[1].p, fb.hi[2].p, fb.id.p,
                                                 fb.node.p, leaf_store.p, leaf_total);
        check_launch("k_scatter");
        k_record<<<grid_for(M, BS), BS, 0, s>>>(M, T, T + M, n_axis.p, n_plane.p, split_rank.p, na.fc.p, leaf_off.p,
                                                leaf_total, na.lo[0].p, na.lo[1].p, na.lo[2].p, na.hi[0].p, na.hi[1].p,
                                                na.hi[2].p, child_start.p, nl.p, cnt.p, tr.kind.p, tr.child.p,
                                                tr.axis.p, tr.plane.p, tr.lo.p, tr.hi.p, tr.leaf_first.p,
                                                tr.leaf_count.p, nb.lo[0].p, nb.lo[1].p, nb.lo[2].p, nb.hi[0].p,
                                                nb.hi[1].p, nb.hi[2].p, nb.fs.p, nb.fc.p);
        check_launch("k_record");
        T += M;
        leaf_total += leaf_frags;
        M = M_next;
        F = F_next;
        std::swap(fa, fb);
        std::swap(na, nb);
        XB_CHECK(depth < 4096, XB_ERR_INTERNAL, "build_regions: runaway recursion");
    }
    level_base.push_back(T);
    // in-order renumbering: counts bottom-up, offsets top-down
    tr.cnt_reg.alloc(T); tr.cnt_ids.alloc(T); tr.off_reg.alloc(T); tr.off_ids.alloc(T);
    int L = (int)level_base.size() - 1;
    for (int l = L - 1; l >= 0; l--) {
        int64_t b = level_base[l], n = level_base[l + 1] - b;
        k_bottom_up<<<grid_for(n, BS), BS, 0, s>>>(b, n, tr.kind.p, tr.child.p, tr.leaf_count.p, tr.cnt_reg.p, tr.cnt_ids.p);
    }
    check_launch("k_bottom_up");
    XB_CUDA(cudaMemsetAsync(tr.off_reg.p, 0, 8, s));
    XB_CUDA(cudaMemsetAsync(tr.off_ids.p, 0, 8, s));
    for (int l = 0; l < L; l++) {
        int64_t b = level_base[l], n = level_base[l + 1] - b;
        k_top_down<<<grid_for(n, BS), BS, 0, s>>>(b, n, tr.kind.p, tr.child.p, tr.cnt_reg.p, tr.cnt_ids.p, tr.off_reg.p, tr.off_ids.p);
    }
    check_launch("k_top_down");
    int64_t R = read_scalar(tr.cnt_reg.p, s);
    int64_t I = read_scalar(tr.cnt_ids.p, s);
    out.n_regions = R;
    out.n_ids = I;
    out.n_kd = T;
    out.kd_depth = L;
    out.kd_level_base = level_base;
    out.kd.alloc(T);
    out.rec.alloc(R ? R : 1);
    out.ids.alloc(I ? I : 1);
    out.lo.alloc(3 * R + 1); out.hi.alloc(3 * R + 1);
    out.brick_off.alloc(R + 1);
    k_finalize<<<grid_for(T, BS), BS, 0, s>>>(T, tr.kind.p, tr.child.p, tr.axis.p, tr.plane.p, tr.lo.p, tr.hi.p,
                                              tr.leaf_first.p, tr.leaf_count.p, tr.off_reg.p, tr.off_ids.p,
                                              leaf_store.p, m.level.p, out.kd.p, out.rec.p, out.ids.p, out.lo.p,
                                              out.hi.p, out.brick_off.p);
    check_launch("k_finalize");
    XB_CUDA(cudaMemcpyAsync(out.brick_off.p + R, &I, 8, cudaMemcpyHostToDevice, s));
    out.vrange.alloc(R * m.n_fields + 1);
    out.vr64.alloc(2 * R * m.n_fields + 1);
    out.finest.alloc(R + 1);
    if (R > 0) {
        k_metadata<<<grid_for(R * 32, BS), BS, 0, s>>>(R, m.n_fields, out.rec.p, out.ids.p, m.lower.p, m.level.p,
                                                       m.dims.p, m.offset.p, m.vals.p, m.n_cells, out.vrange.p,
                                                       out.vr64.p, out.finest.p);
        check_launch("k_metadata");
    }
    XB_CUDA(cudaStreamSynchronize(s));
    build_kd4(out, s);
    out.has_tree = true;
}

}  // namespace xb
