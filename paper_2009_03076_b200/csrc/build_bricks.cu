// build_bricks.cu — GPU brick builder (paper §3.1.2).
//
// Restates `build_bricks` (R/bricks.py:104-228, R/ =
// /root/reference/pkg/src/amrvol/) bit-exactly with level-synchronous kernels:
//   1. validate (alignment, duplicates, octree-ancestor overlaps) — any
//      violation returns XB_ERR_INVALID_CELLS and the host builds the report;
//   2. canonical order: stable LSD radix passes on i, j, k, level
//      (np.lexsort((i, j, k, level)), R/bricks.py:120);
//   3. per tree level: tight node boxes + level range by segmented
//      reductions, leaf / per-cell-leaf / split decision (R/bricks.py:156-202),
//      stable partition `coord[axis] < plane` (R/bricks.py:204);
//   4. in-order renumbering of the leaves (the reference's DFS left-first
//      emission order) and preorder numbering of the split tree;
//   5. brick emission and the x-fastest scalar scatter (R/bricks.py:135-147).
#include "common.cuh"
#include "scan.cuh"
#include <algorithm>

namespace xb {
namespace {

constexpr int BS = 256;

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    return (q * b != a && ((a < 0) != (b < 0))) ? q - 1 : q;
}

__global__ void k_iota(int64_t n, int32_t* a) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) a[t] = (int32_t)t;
}

// key for a stable LSD pass: signed coords flipped to unsigned order
__global__ void k_gather_key(int64_t n, const int32_t* __restrict__ src, const int32_t* __restrict__ perm, int flip,
                             uint32_t* key) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) key[t] = (uint32_t)src[perm[t]] ^ (flip ? 0x80000000u : 0u);
}

__global__ void k_gather_sorted(int64_t n, const int32_t* __restrict__ perm, const int32_t* __restrict__ i,
                                const int32_t* __restrict__ j, const int32_t* __restrict__ k,
                                const int32_t* __restrict__ l, int32_t* si, int32_t* sj, int32_t* sk, int32_t* sl) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int32_t q = perm[t];
    si[t] = i[q]; sj[t] = j[q]; sk[t] = k[q]; sl[t] = l[q];
}

// validation counters: [misaligned, duplicates, overlaps, bad level]
__global__ void k_validate_local(int64_t n, const int32_t* __restrict__ si, const int32_t* __restrict__ sj,
                                 const int32_t* __restrict__ sk, const int32_t* __restrict__ sl, int* counts,
                                 int* level_seen) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int lev = sl[t];
    if (lev < 0 || lev > kMaxLevel) { atomicAdd(&counts[3], 1); return; }
    int64_t m = ((int64_t)1 << lev) - 1;
    if ((si[t] & m) || (sj[t] & m) || (sk[t] & m)) atomicAdd(&counts[0], 1);
    if (t > 0 && si[t] == si[t - 1] && sj[t] == sj[t - 1] && sk[t] == sk[t - 1] && sl[t] == sl[t - 1])
        atomicAdd(&counts[1], 1);
    level_seen[lev] = 1;
}

__device__ __forceinline__ bool kji_less(int32_t k0, int32_t j0, int32_t i0, int32_t k1, int32_t j1, int32_t i1) {
    if (k0 != k1) return k0 < k1;
    if (j0 != j1) return j0 < j1;
    return i0 < i1;
}

// octree ancestor test (R/model.py:420-438): a coarser cell at the ancestor
// anchor of this cell means the two overlap
__global__ void k_validate_overlap(int64_t n, const int32_t* __restrict__ si, const int32_t* __restrict__ sj,
                                   const int32_t* __restrict__ sk, const int32_t* __restrict__ sl,
                                   const int64_t* __restrict__ lvl_start, const int* __restrict__ level_seen,
                                   int* counts) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int lev = sl[t];
    for (int lc = lev + 1; lc <= kMaxLevel; lc++) {
        if (!level_seen[lc]) continue;
        int32_t ai = (int32_t)(((int64_t)si[t] >> lc) << lc), aj = (int32_t)(((int64_t)sj[t] >> lc) << lc),
                ak = (int32_t)(((int64_t)sk[t] >> lc) << lc);
        int64_t lo = lvl_start[lc], hi = lvl_start[lc + 1];
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (kji_less(sk[mid], sj[mid], si[mid], ak, aj, ai)) lo = mid + 1;
            else hi = mid;
        }
        if (lo < lvl_start[lc + 1] && si[lo] == ai && sj[lo] == aj && sk[lo] == ak) atomicAdd(&counts[2], 1);
    }
}

__global__ void k_level_start(int64_t n, const int32_t* __restrict__ sl, int64_t* lvl_start) {
    // lvl_start[l] = first sorted position with level >= l (levels sorted ascending)
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t > n) return;
    int prev = t == 0 ? -1 : sl[t - 1];
    int cur = t == n ? kMaxLevel + 1 : sl[t];
    for (int l = prev + 1; l <= cur && l <= kMaxLevel + 1; l++) lvl_start[l] = t;
}

struct NodeArrays {
    DevBuf<int32_t> lo[3], hi[3], lmin, lmax, fs, fc;
    void ensure(size_t n) {
        for (int a = 0; a < 3; a++) { lo[a].ensure(n); hi[a].ensure(n); }
        lmin.ensure(n); lmax.ensure(n); fs.ensure(n); fc.ensure(n);
    }
};

__global__ void k_node_init(int64_t M, int32_t* lo0, int32_t* lo1, int32_t* lo2, int32_t* hi0, int32_t* hi1,
                            int32_t* hi2, int32_t* lmin, int32_t* lmax) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    lo0[i] = lo1[i] = lo2[i] = INT32_MAX;
    hi0[i] = hi1[i] = hi2[i] = INT32_MIN;
    lmin[i] = INT32_MAX;
    lmax[i] = INT32_MIN;
}

// node_box (R/bricks.py:149-153) + level range, warp-aggregated atomics
__global__ void k_node_reduce(int64_t n, const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                              const int32_t* __restrict__ ck, const int32_t* __restrict__ cl,
                              const int32_t* __restrict__ cnode, int32_t* lo0, int32_t* lo1, int32_t* lo2,
                              int32_t* hi0, int32_t* hi1, int32_t* hi2, int32_t* lmin, int32_t* lmax) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    bool valid = t < n;
    int nd = valid ? cnode[t] : -1;
    int32_t v[8];
    if (valid) {
        int32_t w = 1 << cl[t];
        v[0] = ci[t]; v[1] = cj[t]; v[2] = ck[t];
        v[3] = ci[t] + w; v[4] = cj[t] + w; v[5] = ck[t] + w;
        v[6] = cl[t]; v[7] = cl[t];
    } else {
        v[0] = v[1] = v[2] = v[6] = INT32_MAX;
        v[3] = v[4] = v[5] = v[7] = INT32_MIN;
    }
    const unsigned full = 0xffffffffu;
    int32_t* mins[4] = {lo0, lo1, lo2, lmin};
    int32_t* maxs[4] = {hi0, hi1, hi2, lmax};
    if (warp_uniform(full, nd)) {
        for (int o = 16; o > 0; o >>= 1) {
            v[0] = min(v[0], __shfl_xor_sync(full, v[0], o));
            v[1] = min(v[1], __shfl_xor_sync(full, v[1], o));
            v[2] = min(v[2], __shfl_xor_sync(full, v[2], o));
            v[6] = min(v[6], __shfl_xor_sync(full, v[6], o));
            v[3] = max(v[3], __shfl_xor_sync(full, v[3], o));
            v[4] = max(v[4], __shfl_xor_sync(full, v[4], o));
            v[5] = max(v[5], __shfl_xor_sync(full, v[5], o));
            v[7] = max(v[7], __shfl_xor_sync(full, v[7], o));
        }
        if ((threadIdx.x & 31) == 0 && nd >= 0) {
            atomicMin(&mins[0][nd], v[0]); atomicMin(&mins[1][nd], v[1]); atomicMin(&mins[2][nd], v[2]);
            atomicMin(&mins[3][nd], v[6]);
            atomicMax(&maxs[0][nd], v[3]); atomicMax(&maxs[1][nd], v[4]); atomicMax(&maxs[2][nd], v[5]);
            atomicMax(&maxs[3][nd], v[7]);
        }
    } else if (valid) {
        atomicMin(&mins[0][nd], v[0]); atomicMin(&mins[1][nd], v[1]); atomicMin(&mins[2][nd], v[2]);
        atomicMin(&mins[3][nd], v[6]);
        atomicMax(&maxs[0][nd], v[3]); atomicMax(&maxs[1][nd], v[4]); atomicMax(&maxs[2][nd], v[5]);
        atomicMax(&maxs[3][nd], v[7]);
    }
}

// kind: 0 split, 1 brick leaf, 2 per-cell leaves (R/bricks.py:166-202)
__global__ void k_node_decide(int64_t M, int64_t maxw, const int32_t* lo0, const int32_t* lo1, const int32_t* lo2,
                              const int32_t* hi0, const int32_t* hi1, const int32_t* hi2,
                              const int32_t* __restrict__ lmin, const int32_t* __restrict__ lmax,
                              const int32_t* __restrict__ fc, int32_t* kind, int32_t* axis_o, int32_t* plane_o,
                              int32_t* split /* M+1 */, int32_t* leafc /* M+1 */, int32_t* splitc /* M+1 */,
                              int* err) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    const int64_t cnt = fc[i];
    if (cnt == 0) { atomicAdd(err, 1); kind[i] = 1; split[i] = 0; leafc[i] = 0; splitc[i] = 0; return; }
    const int64_t lo[3] = {lo0[i], lo1[i], lo2[i]}, hi[3] = {hi0[i], hi1[i], hi2[i]};
    const int64_t ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    const int lx = lmax[i];
    const int64_t w = (int64_t)1 << lx;
    const __int128 vol = (__int128)ext[0] * ext[1] * ext[2];
    const __int128 need = (__int128)cnt * w * w * w;
    const bool filled = lmin[i] == lx && need == vol;
    const bool fits = (ext[0] >> lx) <= maxw && (ext[1] >> lx) <= maxw && (ext[2] >> lx) <= maxw;
    int k = 0, axis = 0;
    int64_t plane = 0;
    if (filled && fits) {
        k = 1;
    } else {
        axis = 0;  // argmax, first max
        if (ext[1] > ext[axis]) axis = 1;
        if (ext[2] > ext[axis]) axis = 2;
        const int64_t wc = w, a_lo = lo[axis], a_hi = hi[axis], mid2 = a_lo + a_hi;
        plane = floordiv(mid2 + wc, 2 * wc) * wc;
        if (!(a_lo < plane && plane < a_hi)) {
            const int64_t k_lo = floordiv(a_lo, wc) + 1, k_hi = floordiv(a_hi - 1, wc);
            if (k_lo > k_hi) {
                k = 2;
            } else {
                int64_t km = floordiv(mid2 + wc, 2 * wc);
                km = km < k_lo ? k_lo : (km > k_hi ? k_hi : km);
                plane = km * wc;
            }
        }
    }
    kind[i] = k;
    axis_o[i] = axis;
    plane_o[i] = (int32_t)plane;
    split[i] = k == 0;
    leafc[i] = k == 0 ? 0 : (int32_t)cnt;
    splitc[i] = k == 0 ? (int32_t)cnt : 0;
}

__global__ void k_cell_left(int64_t n, const int32_t* __restrict__ cnode, const int32_t* __restrict__ kind,
                            const int32_t* __restrict__ axis, const int32_t* __restrict__ plane,
                            const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                            const int32_t* __restrict__ ck, int32_t* left) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int nd = cnode[t];
    int l = 0;
    if (kind[nd] == 0) {
        int a = axis[nd];
        int32_t c = a == 0 ? ci[t] : (a == 1 ? cj[t] : ck[t]);
        l = c < plane[nd];
    }
    left[t] = l;
}

__global__ void k_cell_scatter(int64_t n, int64_t tree_base, const int32_t* __restrict__ cnode,
                               const int32_t* __restrict__ kind, const int32_t* __restrict__ fs,
                               const int32_t* __restrict__ fc, const int32_t* __restrict__ sl,
                               const int32_t* __restrict__ child_start, const int32_t* __restrict__ split_rank,
                               const int32_t* __restrict__ leaf_off, int64_t leaf_base, const int32_t* ci,
                               const int32_t* cj, const int32_t* ck, const int32_t* cl, const int32_t* corig,
                               const int32_t* __restrict__ left, int32_t* oi, int32_t* oj, int32_t* ok, int32_t* ol,
                               int32_t* oorig, int32_t* onode, int32_t* leaf_cell, int32_t* leaf_tree) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    int nd = cnode[t];
    int32_t b = fs[nd];
    if (kind[nd] != 0) {
        int64_t q = leaf_base + leaf_off[nd] + (t - b);
        leaf_cell[q] = (int32_t)t;  // index into this level's arrays is stale next level: store orig + coords below
        leaf_tree[q] = (int32_t)(tree_base + nd);
        return;
    }
    int32_t nl = sl[b + fc[nd]] - sl[b];
    int64_t d;
    int32_t child = 2 * split_rank[nd];
    if (left[t]) {
        d = child_start[nd] + (sl[t] - sl[b]);
    } else {
        d = child_start[nd] + nl + ((t - b) - (sl[t] - sl[b]));
        child += 1;
    }
    oi[d] = ci[t]; oj[d] = cj[t]; ok[d] = ck[t]; ol[d] = cl[t]; oorig[d] = corig[t];
    onode[d] = child;
}

// leaves keep their cells' data (coords/level/original row) in leaf storage
__global__ void k_leaf_copy(int64_t n_leaf, const int32_t* __restrict__ leaf_cell, const int32_t* ci, const int32_t* cj,
                            const int32_t* ck, const int32_t* cl, const int32_t* corig, int32_t* li, int32_t* lj,
                            int32_t* lk, int32_t* ll, int32_t* lorig, int64_t base) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n_leaf) return;
    int32_t t = leaf_cell[base + q];
    li[base + q] = ci[t]; lj[base + q] = cj[t]; lk[base + q] = ck[t]; ll[base + q] = cl[t]; lorig[base + q] = corig[t];
}

struct Tree {
    DevBuf<int32_t> kind, child, axis, plane, lo, hi, lmax, leaf_first, leaf_count;
    DevBuf<int64_t> nb, size, boff, pre;
};

__global__ void k_tree_record(int64_t M, int64_t base, int64_t next_base, const int32_t* __restrict__ kind,
                              const int32_t* __restrict__ axis, const int32_t* __restrict__ plane,
                              const int32_t* lo0, const int32_t* lo1, const int32_t* lo2, const int32_t* hi0,
                              const int32_t* hi1, const int32_t* hi2, const int32_t* __restrict__ lmax,
                              const int32_t* __restrict__ fc, const int32_t* __restrict__ split_rank,
                              const int32_t* __restrict__ leaf_off, int64_t leaf_base,
                              const int32_t* __restrict__ child_start, const int32_t* __restrict__ fs,
                              const int32_t* __restrict__ sl, int32_t* t_kind, int32_t* t_child, int32_t* t_axis,
                              int32_t* t_plane, int32_t* t_lo, int32_t* t_hi, int32_t* t_lmax, int32_t* t_lf,
                              int32_t* t_lc, int32_t* nfs, int32_t* nfc) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t g = base + i;
    t_kind[g] = kind[i];
    t_axis[g] = axis[i];
    t_plane[g] = plane[i];
    t_lo[3 * g] = lo0[i]; t_lo[3 * g + 1] = lo1[i]; t_lo[3 * g + 2] = lo2[i];
    t_hi[3 * g] = hi0[i]; t_hi[3 * g + 1] = hi1[i]; t_hi[3 * g + 2] = hi2[i];
    t_lmax[g] = lmax[i];
    if (kind[i] != 0) {
        t_child[g] = -1;
        t_lf[g] = (int32_t)(leaf_base + leaf_off[i]);
        t_lc[g] = fc[i];
        return;
    }
    int32_t c = 2 * split_rank[i];
    t_child[g] = (int32_t)(next_base + c);
    t_lf[g] = 0;
    t_lc[g] = 0;
    int32_t b = fs[i];
    int32_t nl = sl[b + fc[i]] - sl[b];
    nfs[c] = child_start[i];
    nfc[c] = nl;
    nfs[c + 1] = child_start[i] + nl;
    nfc[c + 1] = fc[i] - nl;
}

__global__ void k_tree_up(int64_t base, int64_t M, const int32_t* __restrict__ kind, const int32_t* __restrict__ child,
                          const int32_t* __restrict__ lc, int64_t* nb, int64_t* size) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t g = base + i;
    int k = kind[g];
    if (k == 0) {
        int c = child[g];
        nb[g] = nb[c] + nb[c + 1];
        size[g] = 1 + size[c] + size[c + 1];
    } else {
        nb[g] = k == 1 ? 1 : lc[g];
        size[g] = 1;
    }
}

__global__ void k_tree_down(int64_t base, int64_t M, const int32_t* __restrict__ kind, const int32_t* __restrict__ child,
                            const int64_t* __restrict__ nb, const int64_t* __restrict__ size, int64_t* boff,
                            int64_t* pre) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int64_t g = base + i;
    if (kind[g] != 0) return;
    int c = child[g];
    boff[c] = boff[g];
    boff[c + 1] = boff[g] + nb[c];
    pre[c] = pre[g] + 1;
    pre[c + 1] = pre[g] + 1 + size[c];
}

// brick records; per-cell leaves get one 1x1x1 brick per cell, in order
__global__ void k_emit(int64_t n_leaf_cells, const int32_t* __restrict__ leaf_tree, const int32_t* __restrict__ t_kind,
                       const int32_t* __restrict__ t_lo, const int32_t* __restrict__ t_hi,
                       const int32_t* __restrict__ t_lmax, const int32_t* __restrict__ t_lf,
                       const int64_t* __restrict__ boff, const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                       const int32_t* __restrict__ lk, const int32_t* __restrict__ ll, int32_t* lower, int32_t* level,
                       int32_t* dims, int64_t* cnt /* B+1 */, int32_t* cell_brick) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n_leaf_cells) return;
    int g = leaf_tree[q];
    int k = t_kind[g];
    int64_t rank = q - t_lf[g];
    if (k == 2) {
        int64_t b = boff[g] + rank;
        lower[3 * b] = li[q]; lower[3 * b + 1] = lj[q]; lower[3 * b + 2] = lk[q];
        level[b] = ll[q];
        dims[3 * b] = dims[3 * b + 1] = dims[3 * b + 2] = 1;
        cnt[b] = 1;
        cell_brick[q] = (int32_t)b;
        return;
    }
    int64_t b = boff[g];
    cell_brick[q] = (int32_t)b;
    if (rank != 0) return;
    int lx = t_lmax[g];
    int64_t c = 1;
    for (int a = 0; a < 3; a++) {
        lower[3 * b + a] = t_lo[3 * g + a];
        int32_t d = (t_hi[3 * g + a] - t_lo[3 * g + a]) >> lx;
        dims[3 * b + a] = d;
        c *= d;
    }
    level[b] = lx;
    cnt[b] = c;
}

__global__ void k_scatter_values(int64_t n_leaf_cells, int F, int64_t N, const int32_t* __restrict__ cell_brick,
                                 const int32_t* __restrict__ lower, const int32_t* __restrict__ level,
                                 const int32_t* __restrict__ dims, const int64_t* __restrict__ offset,
                                 const int32_t* __restrict__ li, const int32_t* __restrict__ lj,
                                 const int32_t* __restrict__ lk, const int32_t* __restrict__ lorig,
                                 const float* __restrict__ values /* (n, F) */, float* vals /* (F, N) */) {
    int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n_leaf_cells) return;
    int b = cell_brick[q];
    int lev = level[b];
    int64_t gx = ((int64_t)li[q] - lower[3 * b]) >> lev;
    int64_t gy = ((int64_t)lj[q] - lower[3 * b + 1]) >> lev;
    int64_t gz = ((int64_t)lk[q] - lower[3 * b + 2]) >> lev;
    int64_t slot = gx + (int64_t)dims[3 * b] * (gy + (int64_t)dims[3 * b + 1] * gz);
    int64_t row = lorig[q];
    for (int f = 0; f < F; f++) vals[f * N + offset[b] + slot] = values[row * F + f];
}

__global__ void k_split_tree(int64_t T, const int32_t* __restrict__ kind, const int32_t* __restrict__ child,
                             const int32_t* __restrict__ axis, const int32_t* __restrict__ plane,
                             const int32_t* __restrict__ t_lo, const int32_t* __restrict__ t_hi,
                             const int32_t* __restrict__ t_lmax, const int64_t* __restrict__ nb,
                             const int64_t* __restrict__ boff, const int64_t* __restrict__ pre, int32_t* o_axis,
                             double* o_pos, int32_t* o_left, int32_t* o_right, int32_t* o_bs, int32_t* o_bc,
                             double* o_lo, double* o_hi, double* o_mh) {
    int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (g >= T) return;
    int64_t p = pre[g];
    int k = kind[g];
    for (int a = 0; a < 3; a++) {
        o_lo[3 * p + a] = (double)t_lo[3 * g + a];
        o_hi[3 * p + a] = (double)t_hi[3 * g + a];
    }
    o_mh[p] = 0.5 * ldexp(1.0, t_lmax[g]);
    if (k == 0) {
        o_axis[p] = axis[g];
        o_pos[p] = (double)plane[g];
        o_left[p] = (int32_t)pre[child[g]];
        o_right[p] = (int32_t)pre[child[g] + 1];
        o_bs[p] = 0;
        o_bc[p] = 0;
    } else {
        o_axis[p] = -1;
        o_pos[p] = 0.0;
        o_left[p] = 0;
        o_right[p] = 0;
        o_bs[p] = (int32_t)boff[g];
        o_bc[p] = (int32_t)nb[g];
    }
}

__global__ void k_pack_bricks(int64_t B, const int32_t* __restrict__ lower, const int32_t* __restrict__ level,
                              const int32_t* __restrict__ dims, const int64_t* __restrict__ offset, int4* ba,
                              uint32_t* bm) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    ba[b] = make_int4(lower[3 * b], lower[3 * b + 1], lower[3 * b + 2], (int32_t)(uint32_t)offset[b]);
    bm[b] = pack_brick_meta(level[b], dims[3 * b], dims[3 * b + 1], dims[3 * b + 2]);
}

}  // namespace

// Finish a DevModel whose lower/level/dims/offset/vals are set: packed
// records + range metadata.  Used by the builder and by host uploads.
void finish_model(DevModel& m, cudaStream_t s) {
    const int64_t B = m.n_bricks;
    m.brick_a.alloc(B + 1);
    m.brick_m.alloc(B + 1);
    m.coord_min = 0;
    m.coord_max = 0;
    m.max_level = 0;
    if (B == 0) return;
    XB_CHECK(m.n_cells < (1ll << 32), XB_ERR_RANGE, "more than 2^32 cells are not supported by the packed layout");
    auto lower = m.lower.to_host(3 * B, s);
    auto level = m.level.to_host(B, s);
    auto dims = m.dims.to_host(3 * B, s);
    int64_t cmin = INT64_MAX, cmax = INT64_MIN;
    int lmax = 0;
    for (int64_t b = 0; b < B; b++) {
        XB_CHECK(level[b] >= 0 && level[b] <= kMaxLevel, XB_ERR_RANGE, "brick level out of range");
        lmax = std::max(lmax, level[b]);
        for (int a = 0; a < 3; a++) {
            XB_CHECK(dims[3 * b + a] >= 1 && dims[3 * b + a] <= kMaxDim, XB_ERR_RANGE, "brick dims out of range (1..511)");
            int64_t lo = lower[3 * b + a], hi = lo + ((int64_t)dims[3 * b + a] << level[b]);
            cmin = std::min(cmin, lo);
            cmax = std::max(cmax, hi);
        }
    }
    XB_CHECK(cmin > -(1ll << 30) && cmax < (1ll << 30), XB_ERR_RANGE, "brick coordinates exceed +-2^30");
    m.coord_min = (int32_t)cmin;
    m.coord_max = (int32_t)cmax;
    m.max_level = lmax;
    k_pack_bricks<<<grid_for(B, BS), BS, 0, s>>>(B, m.lower.p, m.level.p, m.dims.p, m.offset.p, m.brick_a.p, m.brick_m.p);
    check_launch("k_pack_bricks");
    XB_CUDA(cudaStreamSynchronize(s));
}

// returns false (and leaves `m` empty) if the cells fail validation
bool build_bricks_device(const int32_t* hi_, const int32_t* hj, const int32_t* hk, const int32_t* hl, const float* hv,
                         int64_t n, int F, int64_t maxw, bool keep_tree, int device, DevModel& m, cudaStream_t s) {
    DeviceGuard guard(device);
    m = DevModel();
    m.device = device;
    m.n_fields = F;
    XB_CHECK(n < (1ll << 31) - 2, XB_ERR_RANGE, "build_bricks: more than 2^31 cells");
    XB_CHECK(maxw >= 1, XB_ERR_ARG, "max_brick_width must be >= 1");
    if (n == 0) {
        m.offset.alloc(1);
        XB_CUDA(cudaMemsetAsync(m.offset.p, 0, 8, s));
        m.vals.alloc(1);
        finish_model(m, s);
        return true;
    }
    CubTemp tmp;
    DevBuf<int32_t> di, dj, dk, dl;
    di.upload(hi_, n, s); dj.upload(hj, n, s); dk.upload(hk, n, s); dl.upload(hl, n, s);
    DevBuf<float> dv;
    dv.upload(hv, n * F, s);
    // ---- canonical order: lexsort((i, j, k, level)) = LSD passes i, j, k, level
    DevBuf<int32_t> perm(n), perm2(n);
    DevBuf<uint32_t> key(n), key2(n);
    k_iota<<<grid_for(n, BS), BS, 0, s>>>(n, perm.p);
    const int32_t* src[4] = {di.p, dj.p, dk.p, dl.p};
    for (int pass = 0; pass < 4; pass++) {
        k_gather_key<<<grid_for(n, BS), BS, 0, s>>>(n, src[pass], perm.p, pass < 3, key.p);
        sort_pairs(tmp, key.p, key2.p, perm.p, perm2.p, n, 0, 32, s);
        std::swap(perm, perm2);
    }
    check_launch("lexsort");
    DevBuf<int32_t> ci(n), cj(n), ck(n), cl(n);
    k_gather_sorted<<<grid_for(n, BS), BS, 0, s>>>(n, perm.p, di.p, dj.p, dk.p, dl.p, ci.p, cj.p, ck.p, cl.p);
    // ---- validation (R/model.py:392-457; report built on the host on failure)
    DevBuf<int> counts(4), seen(kMaxLevel + 2);
    XB_CUDA(cudaMemsetAsync(counts.p, 0, 4 * sizeof(int), s));
    XB_CUDA(cudaMemsetAsync(seen.p, 0, (kMaxLevel + 2) * sizeof(int), s));
    k_validate_local<<<grid_for(n, BS), BS, 0, s>>>(n, ci.p, cj.p, ck.p, cl.p, counts.p, seen.p);
    check_launch("k_validate_local");
    auto c4 = counts.to_host(4, s);
    if (c4[0] || c4[1] || c4[3]) return false;
    DevBuf<int64_t> lvl_start(kMaxLevel + 3);
    k_level_start<<<grid_for(n + 1, BS), BS, 0, s>>>(n, cl.p, lvl_start.p);
    k_validate_overlap<<<grid_for(n, BS), BS, 0, s>>>(n, ci.p, cj.p, ck.p, cl.p, lvl_start.p, seen.p, counts.p);
    check_launch("k_validate_overlap");
    c4 = counts.to_host(4, s);
    if (c4[2]) return false;
    {   // anchors + widths must fit int32 for the node boxes (R/model.py keeps int64)
        DevBuf<int32_t> r1;
        const int32_t lmx = reduce_max(tmp, cl.p, n, r1, s);
        int64_t lo = INT64_MAX, hi = INT64_MIN;
        for (const int32_t* a : {ci.p, cj.p, ck.p}) {
            lo = std::min<int64_t>(lo, reduce_min(tmp, a, n, r1, s));
            hi = std::max<int64_t>(hi, reduce_max(tmp, a, n, r1, s));
        }
        XB_CHECK(lo > -(1ll << 30) && hi + (1ll << lmx) < (1ll << 30), XB_ERR_RANGE,
                 "build_bricks: cell coordinates exceed +-2^30");
    }
    // ---- level loop
    DevBuf<int32_t> corig(n), cnode(n);
    XB_CUDA(cudaMemcpyAsync(corig.p, perm.p, n * 4, cudaMemcpyDeviceToDevice, s));
    XB_CUDA(cudaMemsetAsync(cnode.p, 0, n * 4, s));
    DevBuf<int32_t> ni(n), nj(n), nk(n), nlv(n), norig(n), nnode(n);
    NodeArrays na, nb2;
    na.ensure(1);
    int32_t zero = 0, n32 = (int32_t)n;
    XB_CUDA(cudaMemcpyAsync(na.fs.p, &zero, 4, cudaMemcpyHostToDevice, s));
    XB_CUDA(cudaMemcpyAsync(na.fc.p, &n32, 4, cudaMemcpyHostToDevice, s));
    Tree tr;
    DevBuf<int32_t> leaf_cell(n), leaf_tree(n), li(n), lj(n), lk(n), ll(n), lorig(n);
    DevBuf<int32_t> kind, axis, plane, split, leafc, splitc, split_rank, leaf_off, child_start, left, sl;
    DevBuf<int> err(1);
    XB_CUDA(cudaMemsetAsync(err.p, 0, sizeof(int), s));
    std::vector<int64_t> level_base;
    int64_t T = 0, leaf_total = 0, M = 1, cells = n;
    while (M > 0) {
        level_base.push_back(T);
        k_node_init<<<grid_for(M, BS), BS, 0, s>>>(M, na.lo[0].p, na.lo[1].p, na.lo[2].p, na.hi[0].p, na.hi[1].p,
                                                   na.hi[2].p, na.lmin.p, na.lmax.p);
        k_node_reduce<<<grid_for(cells, BS), BS, 0, s>>>(cells, ci.p, cj.p, ck.p, cl.p, cnode.p, na.lo[0].p,
                                                         na.lo[1].p, na.lo[2].p, na.hi[0].p, na.hi[1].p,
                                                         na.hi[2].p, na.lmin.p, na.lmax.p);
        kind.ensure(M); axis.ensure(M); plane.ensure(M); split.ensure(M + 1); leafc.ensure(M + 1); splitc.ensure(M + 1);
        split_rank.ensure(M + 1); leaf_off.ensure(M + 1); child_start.ensure(M + 1);
        k_node_decide<<<grid_for(M, BS), BS, 0, s>>>(M, maxw, na.lo[0].p, na.lo[1].p, na.lo[2].p, na.hi[0].p,
                                                     na.hi[1].p, na.hi[2].p, na.lmin.p, na.lmax.p, na.fc.p, kind.p,
                                                     axis.p, plane.p, split.p, leafc.p, splitc.p, err.p);
        check_launch("k_node_decide");
        XB_CUDA(cudaMemsetAsync(split.p + M, 0, 4, s));
        XB_CUDA(cudaMemsetAsync(leafc.p + M, 0, 4, s));
        XB_CUDA(cudaMemsetAsync(splitc.p + M, 0, 4, s));
        exclusive_sum(tmp, split.p, split_rank.p, M + 1, s);
        exclusive_sum(tmp, leafc.p, leaf_off.p, M + 1, s);
        exclusive_sum(tmp, splitc.p, child_start.p, M + 1, s);
        left.ensure(cells + 1);
        sl.ensure(cells + 1);
        k_cell_left<<<grid_for(cells, BS), BS, 0, s>>>(cells, cnode.p, kind.p, axis.p, plane.p, ci.p, cj.p, ck.p, left.p);
        XB_CUDA(cudaMemsetAsync(left.p + cells, 0, 4, s));
        exclusive_sum(tmp, left.p, sl.p, cells + 1, s);
        int32_t n_split = read_scalar(split_rank.p + M, s);
        int32_t n_leafc = read_scalar(leaf_off.p + M, s);
        int32_t cells_next = read_scalar(child_start.p + M, s);
        int64_t M_next = 2 * (int64_t)n_split;
        k_cell_scatter<<<grid_for(cells, BS), BS, 0, s>>>(cells, T, cnode.p, kind.p, na.fs.p, na.fc.p, sl.p,
                                                          child_start.p, split_rank.p, leaf_off.p, leaf_total, ci.p,
                                                          cj.p, ck.p, cl.p, corig.p, left.p, ni.p, nj.p, nk.p,
                                                          nlv.p, norig.p, nnode.p, leaf_cell.p, leaf_tree.p);
        check_launch("k_cell_scatter");
        if (n_leafc > 0)
            k_leaf_copy<<<grid_for(n_leafc, BS), BS, 0, s>>>(n_leafc, leaf_cell.p, ci.p, cj.p, ck.p, cl.p, corig.p, li.p,
                                                             lj.p, lk.p, ll.p, lorig.p, leaf_total);
        size_t Tn = T + M;
        grow_keep(tr.kind, Tn, T, s); grow_keep(tr.child, Tn, T, s); grow_keep(tr.axis, Tn, T, s);
        grow_keep(tr.plane, Tn, T, s); grow_keep(tr.lo, 3 * Tn, 3 * T, s); grow_keep(tr.hi, 3 * Tn, 3 * T, s);
        grow_keep(tr.lmax, Tn, T, s); grow_keep(tr.leaf_first, Tn, T, s); grow_keep(tr.leaf_count, Tn, T, s);
        nb2.ensure(M_next > 0 ? M_next : 1);
        k_tree_record<<<grid_for(M, BS), BS, 0, s>>>(M, T, T + M, kind.p, axis.p, plane.p, na.lo[0].p, na.lo[1].p,
                                                     na.lo[2].p, na.hi[0].p, na.hi[1].p, na.hi[2].p, na.lmax.p,
                                                     na.fc.p, split_rank.p, leaf_off.p, leaf_total, child_start.p,
                                                     na.fs.p, sl.p, tr.kind.p, tr.child.p, tr.axis.p, tr.plane.p,
                                                     tr.lo.p, tr.hi.p, tr.lmax.p, tr.leaf_first.p, tr.leaf_count.p,
                                                     nb2.fs.p, nb2.fc.p);
        check_launch("k_tree_record");
        T += M;
        leaf_total += n_leafc;
        M = M_next;
        cells = cells_next;
        std::swap(ci, ni); std::swap(cj, nj); std::swap(ck, nk); std::swap(cl, nlv); std::swap(corig, norig);
        std::swap(cnode, nnode);
        std::swap(na, nb2);
        XB_CHECK(level_base.size() < 100000, XB_ERR_INTERNAL, "build_bricks: runaway recursion");
    }
    level_base.push_back(T);
    XB_CHECK(read_scalar(err.p, s) == 0, XB_ERR_INTERNAL, "build_bricks: empty k-d node");
    XB_CHECK(leaf_total == n, XB_ERR_INTERNAL, "build_bricks: leaf cells != input cells");
    // ---- renumbering
    tr.nb.alloc(T); tr.size.alloc(T); tr.boff.alloc(T); tr.pre.alloc(T);
    const int L = (int)level_base.size() - 1;
    for (int l = L - 1; l >= 0; l--) {
        int64_t b = level_base[l], cnt = level_base[l + 1] - b;
        k_tree_up<<<grid_for(cnt, BS), BS, 0, s>>>(b, cnt, tr.kind.p, tr.child.p, tr.leaf_count.p, tr.nb.p, tr.size.p);
    }
    XB_CUDA(cudaMemsetAsync(tr.boff.p, 0, 8, s));
    XB_CUDA(cudaMemsetAsync(tr.pre.p, 0, 8, s));
    for (int l = 0; l < L; l++) {
        int64_t b = level_base[l], cnt = level_base[l + 1] - b;
        k_tree_down<<<grid_for(cnt, BS), BS, 0, s>>>(b, cnt, tr.kind.p, tr.child.p, tr.nb.p, tr.size.p, tr.boff.p, tr.pre.p);
    }
    check_launch("tree renumbering");
    const int64_t B = read_scalar(tr.nb.p, s);
    m.n_bricks = B;
    m.lower.alloc(3 * B); m.level.alloc(B); m.dims.alloc(3 * B); m.offset.alloc(B + 1);
    DevBuf<int64_t> bcnt(B + 1);
    DevBuf<int32_t> cell_brick(n);
    XB_CUDA(cudaMemsetAsync(bcnt.p + B, 0, 8, s));
    k_emit<<<grid_for(n, BS), BS, 0, s>>>(n, leaf_tree.p, tr.kind.p, tr.lo.p, tr.hi.p, tr.lmax.p, tr.leaf_first.p,
                                          tr.boff.p, li.p, lj.p, lk.p, ll.p, m.lower.p, m.level.p, m.dims.p, bcnt.p,
                                          cell_brick.p);
    check_launch("k_emit");
    exclusive_sum(tmp, bcnt.p, m.offset.p, B + 1, s);
    m.n_cells = read_scalar(m.offset.p + B, s);
    XB_CHECK(m.n_cells == n, XB_ERR_INTERNAL, "build_bricks: bricks do not tile the cells");
    m.vals.alloc(F * n + 1);
    k_scatter_values<<<grid_for(n, BS), BS, 0, s>>>(n, F, n, cell_brick.p, m.lower.p, m.level.p, m.dims.p, m.offset.p,
                                                    li.p, lj.p, lk.p, lorig.p, dv.p, m.vals.p);
    check_launch("k_scatter_values");
    if (keep_tree) {
        m.n_tree = T;
        m.t_axis.alloc(T); m.t_left.alloc(T); m.t_right.alloc(T); m.t_bstart.alloc(T); m.t_bcount.alloc(T);
        m.t_pos.alloc(T); m.t_lo.alloc(3 * T); m.t_hi.alloc(3 * T); m.t_mh.alloc(T);
        k_split_tree<<<grid_for(T, BS), BS, 0, s>>>(T, tr.kind.p, tr.child.p, tr.axis.p, tr.plane.p, tr.lo.p, tr.hi.p,
                                                    tr.lmax.p, tr.nb.p, tr.boff.p, tr.pre.p, m.t_axis.p, m.t_pos.p,
                                                    m.t_left.p, m.t_right.p, m.t_bstart.p, m.t_bcount.p, m.t_lo.p,
                                                    m.t_hi.p, m.t_mh.p);
        check_launch("k_split_tree");
    }
    finish_model(m, s);
    return true;
}

}  // namespace xb
