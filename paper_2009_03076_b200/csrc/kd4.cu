// kd4.cu — collapse the region k-d tree (BFS order, build_regions.cu) into
// 4-ary nodes of two binary levels each, and fold an active set's per-node
// flags into per-slot masks.  The warp traversal (render.cu:k_warp) expands a
// Kd4 node into up to four ordered children with the same exact, conservative
// slab arithmetic as the binary walk; leaves are resolved from the parent's
// child codes without loading them.  Halving the depth halves the dependent
// node loads per ray.
#include "accel.cuh"
#include "scan.cuh"

namespace xb {
namespace {

__device__ __forceinline__ bool kd_interior(KdNode n) { return n.a != -1 && (n.a & 3) != 3; }
__device__ __forceinline__ int kd_leaf_code(KdNode n) { return n.a == -1 ? -1 : -2 - (n.a >> 2); }

__global__ void k_kd4_mark(int64_t base, int64_t n, const KdNode* __restrict__ kd, int32_t* mark) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) mark[base + i] = kd_interior(kd[base + i]) ? 1 : 0;
}

__global__ void k_kd4_fill(int64_t base, int64_t n, const KdNode* __restrict__ kd, const int32_t* __restrict__ idx,
                           Kd4Node* __restrict__ out, int4* __restrict__ bin) {
    const int64_t i = base + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= base + n) return;
    const KdNode nd = kd[i];
    if (!kd_interior(nd)) return;
    Kd4Node o;
    int bn[4];
    o.plane[0] = nd.b;
    uint32_t axes = (uint32_t)(nd.a & 3);
    const int left = nd.a >> 2;
    for (int side = 0; side < 2; side++) {
        const int c = left + side;
        const KdNode cn = kd[c];
        if (kd_interior(cn)) {
            axes |= (uint32_t)(cn.a & 3) << (2 + 2 * side);
            o.plane[1 + side] = cn.b;
            const int g = cn.a >> 2;
            for (int q = 0; q < 2; q++) {
                const KdNode gn = kd[g + q];
                o.child[2 * side + q] = kd_interior(gn) ? idx[g + q] : kd_leaf_code(gn);
                bn[2 * side + q] = g + q;
            }
        } else {
            axes |= 3u << (2 + 2 * side);
            o.plane[1 + side] = 0;
            o.child[2 * side] = kd_leaf_code(cn);
            o.child[2 * side + 1] = -1;
            bn[2 * side] = c;
            bn[2 * side + 1] = -1;
        }
    }
    o.axes = axes;
    const int k = idx[i];
    out[k] = o;
    bin[k] = make_int4(bn[0], bn[1], bn[2], bn[3]);
}

__global__ void k_kd4_mask(int64_t n, const int4* __restrict__ bin, const uint8_t* __restrict__ flags,
                           uint8_t* __restrict__ mask) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int4 b = bin[i];
    uint8_t m = 0;
    if (b.x >= 0 && flags[b.x]) m |= 1;
    if (b.y >= 0 && flags[b.y]) m |= 2;
    if (b.z >= 0 && flags[b.z]) m |= 4;
    if (b.w >= 0 && flags[b.w]) m |= 8;
    mask[i] = m;
}

}  // namespace

void build_kd4(DevRegions& R, cudaStream_t s) {
    const int64_t T = R.n_kd;
    const auto& lb = R.kd_level_base;
    R.n_kd4 = 0;
    if (T == 0 || lb.size() < 2) {
        R.kd4.alloc(1);
        R.kd4_bin.alloc(1);
        return;
    }
    const int BS = 256;
    DevBuf<int32_t> mark(T + 1), idx(T + 1);
    XB_CUDA(cudaMemsetAsync(mark.p, 0, (T + 1) * sizeof(int32_t), s));
    for (size_t l = 0; l + 1 < lb.size(); l += 2) {  // Kd4 nodes: interior nodes on even binary levels
        const int64_t b = lb[l], m = lb[l + 1] - b;
        if (m > 0) k_kd4_mark<<<grid_for(m, BS), BS, 0, s>>>(b, m, R.kd.p, mark.p);
    }
    check_launch("k_kd4_mark");
    CubTemp tmp;
    exclusive_sum(tmp, mark.p, idx.p, T + 1, s);
    R.n_kd4 = read_scalar(idx.p + T, s);
    R.kd4.alloc(R.n_kd4 + 1);
    R.kd4_bin.alloc(R.n_kd4 + 1);
    for (size_t l = 0; l + 1 < lb.size(); l += 2) {
        const int64_t b = lb[l], m = lb[l + 1] - b;
        if (m > 0) k_kd4_fill<<<grid_for(m, BS), BS, 0, s>>>(b, m, R.kd.p, idx.p, R.kd4.p, R.kd4_bin.p);
    }
    check_launch("k_kd4_fill");
    XB_CUDA(cudaStreamSynchronize(s));
}

void build_kd4_mask(const DevRegions& R, const uint8_t* flags, DevBuf<uint8_t>& mask, cudaStream_t s) {
    mask.alloc_async(R.n_kd4 + 1, s);
    XB_CUDA(cudaMemsetAsync(mask.p, 0, R.n_kd4 + 1, s));
    if (R.n_kd4 > 0) k_kd4_mask<<<grid_for(R.n_kd4, 256), 256, 0, s>>>(R.n_kd4, R.kd4_bin.p, flags, mask.p);
    check_launch("k_kd4_mask");
}

}  // namespace xb
