// lbvh.cu — GPU LBVH build over active region boxes (lbvh.cuh):
//   1. 63-bit Morton code of each box centre (21 bits per axis, exact integer
//      arithmetic on half-unit corners, normalised to the region-set bounds);
//   2. CUB radix sort of (code, region id);
//   3. Karras 2012: every internal node finds its key range and split from
//      common-prefix lengths (equal codes break ties on the sorted index);
//   4. bottom-up refit with per-node arrival counters: the second child to
//      arrive forms the exact int32 union box and the subtree height.
#include <algorithm>
#include <chrono>
#include "lbvh.cuh"
#include "scan.cuh"

namespace xb {
namespace {

constexpr int BS = 256;

__device__ __forceinline__ uint64_t spread21(uint64_t v) {
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__global__ void k_morton(int64_t n, const int32_t* __restrict__ prims, const RegionRec* __restrict__ rec, int3 cmin,
                         int3 cext, uint64_t* __restrict__ key, int32_t* __restrict__ val) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int r = prims[i];
    const RegionRec rr = rec[r];
    const int64_t c[3] = {(int64_t)rr.lo[0] + rr.hi[0], (int64_t)rr.lo[1] + rr.hi[1], (int64_t)rr.lo[2] + rr.hi[2]};
    const int64_t mn[3] = {cmin.x, cmin.y, cmin.z}, ex[3] = {cext.x, cext.y, cext.z};
    uint64_t q[3];
    for (int a = 0; a < 3; a++) {
        int64_t v = ((c[a] - mn[a]) * 0x1fffff) / (ex[a] > 0 ? ex[a] : 1);
        q[a] = (uint64_t)(v < 0 ? 0 : (v > 0x1fffff ? 0x1fffff : v));
    }
    key[i] = spread21(q[0]) | spread21(q[1]) << 1 | spread21(q[2]) << 2;
    val[i] = r;
}

__device__ __forceinline__ int delta(const uint64_t* __restrict__ k, int64_t n, int64_t i, int64_t j) {
    if (j < 0 || j >= n) return -1;
    const uint64_t a = k[i], b = k[j];
    if (a == b) return 64 + __clzll((long long)(i ^ j));
    return __clzll((long long)(a ^ b));
}

__global__ void k_karras(int64_t n, const uint64_t* __restrict__ k, LbvhNode* __restrict__ nodes,
                         int32_t* __restrict__ parent_int, int32_t* __restrict__ parent_leaf) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n - 1) return;
    const int d = delta(k, n, i, i + 1) - delta(k, n, i, i - 1) >= 0 ? 1 : -1;
    const int dmin = delta(k, n, i, i - d);
    int64_t lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin) lmax *= 2;
    int64_t l = 0;
    for (int64_t t = lmax / 2; t >= 1; t /= 2)
        if (delta(k, n, i, i + (l + t) * d) > dmin) l += t;
    const int64_t j = i + l * d;
    const int dnode = delta(k, n, i, j);
    int64_t s = 0, div = 2;
    for (;;) {
        const int64_t t = (l + div - 1) / div;
        if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
        if (t <= 1) break;
        div *= 2;
    }
    const int64_t g = i + s * d + (d < 0 ? -1 : 0);
    const int64_t lo = i < j ? i : j, hi = i < j ? j : i;
    const int32_t left = lo == g ? ~(int32_t)g : (int32_t)g;
    const int32_t right = hi == g + 1 ? ~(int32_t)(g + 1) : (int32_t)(g + 1);
    nodes[i].left = left;
    nodes[i].right = right;
    if (left < 0) parent_leaf[~left] = (int32_t)i; else parent_int[left] = (int32_t)i;
    if (right < 0) parent_leaf[~right] = (int32_t)i; else parent_int[right] = (int32_t)i;
}

__global__ void k_refit(int64_t n, const int32_t* __restrict__ prims, const RegionRec* __restrict__ rec,
                        LbvhNode* nodes, const int32_t* __restrict__ parent_int, const int32_t* __restrict__ parent_leaf,
                        int32_t* visits, int32_t* height) {
    const int64_t kidx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (kidx >= n) return;
    int32_t node = parent_leaf[kidx];
    while (node >= 0) {
        __threadfence();
        if (atomicAdd(&visits[node], 1) == 0) return;  // the sibling subtree is not finished yet
        __threadfence();
        volatile LbvhNode* vn = nodes;
        const int32_t c[2] = {vn[node].left, vn[node].right};
        int32_t lo[3] = {INT32_MAX, INT32_MAX, INT32_MAX}, hi[3] = {INT32_MIN, INT32_MIN, INT32_MIN};
        int h = 0;
        for (int q = 0; q < 2; q++) {
            if (c[q] < 0) {
                const RegionRec& rr = rec[prims[~c[q]]];
                for (int a = 0; a < 3; a++) {
                    lo[a] = min(lo[a], rr.lo[a]);
                    hi[a] = max(hi[a], rr.hi[a]);
                }
            } else {
                for (int a = 0; a < 3; a++) {
                    lo[a] = min(lo[a], vn[c[q]].lo[a]);
                    hi[a] = max(hi[a], vn[c[q]].hi[a]);
                }
                h = max(h, ((volatile int32_t*)height)[c[q]]);
            }
        }
        for (int a = 0; a < 3; a++) {
            vn[node].lo[a] = lo[a];
            vn[node].hi[a] = hi[a];
        }
        ((volatile int32_t*)height)[node] = h + 1;
        node = parent_int[node];
    }
}

}  // namespace

void build_lbvh(const DevRegions& R, const int32_t* prims_in, int64_t n, DevLbvh& out, cudaStream_t s) {
    const auto t0 = std::chrono::steady_clock::now();
    out = DevLbvh();
    out.n_prims = n;
    out.prims.alloc(n + 1);
    out.nodes.alloc(std::max<int64_t>(n - 1, 1));
    if (n == 0) return;
    const int3 cmin = make_int3(2 * R.root_lo[0], 2 * R.root_lo[1], 2 * R.root_lo[2]);
    const int3 cext = make_int3(2 * (R.root_hi[0] - R.root_lo[0]), 2 * (R.root_hi[1] - R.root_lo[1]),
                                2 * (R.root_hi[2] - R.root_lo[2]));
    DevBuf<uint64_t> key(n), key2(n);
    DevBuf<int32_t> val(n);
    k_morton<<<grid_for(n, BS), BS, 0, s>>>(n, prims_in, R.rec.p, cmin, cext, key.p, val.p);
    check_launch("k_morton");
    CubTemp tmp;
    sort_pairs(tmp, key.p, key2.p, val.p, out.prims.p, n, 0, 63, s);
    if (n == 1) {
        out.depth = 0;
        XB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    DevBuf<int32_t> parent_int(n), parent_leaf(n), visits(n), height(n);
    XB_CUDA(cudaMemsetAsync(visits.p, 0, n * sizeof(int32_t), s));
    XB_CUDA(cudaMemsetAsync(height.p, 0, n * sizeof(int32_t), s));
    XB_CUDA(cudaMemsetAsync(parent_int.p, 0xff, sizeof(int32_t), s));  // root: no parent
    k_karras<<<grid_for(n - 1, BS), BS, 0, s>>>(n, key2.p, out.nodes.p, parent_int.p, parent_leaf.p);
    check_launch("k_karras");
    k_refit<<<grid_for(n, BS), BS, 0, s>>>(n, out.prims.p, R.rec.p, out.nodes.p, parent_int.p, parent_leaf.p,
                                           visits.p, height.p);
    check_launch("k_refit");
    out.depth = read_scalar(height.p, s);  // root height = deepest leaf depth
    XB_CHECK(out.depth + 2 < kLbvhStack, XB_ERR_RANGE, "LBVH deeper than the traversal stack");
    out.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace xb
