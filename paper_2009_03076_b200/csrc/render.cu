// render.cu — the fused sm_100a ray-march kernel (paper §4-5) and the
// single-ray batch kernel behind integrate_ray / iso_intersect.
//
// One thread per pixel; a CUDA block renders one 16x8 screen tile, each warp
// an 8x4 sub-tile (coherent rays share regions and bricks in L1).  Per pixel:
// ray setup, rho hash, clip planes, optional iso pass, volume pass over the
// ordered k-d region walk, iso composite, RGBA8 quantisation — the body of
// `_render_kernel` (R/render.py:521-578).  The transfer function (8 KB of
// doubles) travels in the kernel parameter block and is staged in shared
// memory.  Tiles are dealt round-robin over ranks (multi-GPU screen tiling,
// SURVEY.md §8(e)); the global pixel index feeds the rho hash so every rank
// renders exactly the pixels a single GPU would.
#include "march.cuh"
#include "render.cuh"

namespace xb {

template <int GRAD, bool ISO, bool COUNT>
__global__ void __launch_bounds__(kTileW* kTileH) k_render(const __grid_constant__ RenderArgs A) {
    __shared__ double s_tf[1024];
    __shared__ unsigned long long s_stats[3];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = A.tf[i];
    if (threadIdx.x < 3) s_stats[threadIdx.x] = 0;
    __syncthreads();

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int lx = (warp & 1) * 8 + (lane & 7);      // warp = 8x4 pixels
    const int ly = (warp >> 1) * 4 + (lane >> 3);
    const int64_t tile = (int64_t)A.tile_rank + (int64_t)blockIdx.x * A.tile_world;
    const int tx = (int)(tile % A.tiles_x), ty = (int)(tile / A.tiles_x);
    const int x = tx * kTileW + lx, y = ty * kTileH + ly;
    const bool live = tile < (int64_t)A.tiles_x * A.tiles_y && x < A.W && y < A.H;

    RayStats st = {0, 0, 0};
    if (live) {
        const int64_t pix = (int64_t)y * A.W + x;
        const double sx = (2.0 * ((double)x + 0.5) / (double)A.W - 1.0) * A.tan_half * A.aspect;
        const double sy = (1.0 - 2.0 * ((double)y + 0.5) / (double)A.H) * A.tan_half;
        Ray r;
#pragma unroll
        for (int a = 0; a < 3; a++) r.d[a] = A.fwd[a] + sx * A.right[a] + sy * A.up[a];
        const double inv = 1.0 / sqrt(r.d[0] * r.d[0] + r.d[1] * r.d[1] + r.d[2] * r.d[2]);
#pragma unroll
        for (int a = 0; a < 3; a++) {
            r.d[a] *= inv;
            r.o[a] = A.pos[a];
            r.inv[a] = 1.0 / r.d[a];
        }
        const double rho = rho_hash((uint64_t)pix, A.M.seed);
        double tmin = 0.0, tmax = kTFar;
        clip_ray(A.M, r, tmin, tmax);
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        if (tmin < tmax) {
            double t_end = tmax, g[3] = {0.0, 0.0, 0.0}, t_hit = 0.0;
            bool hit = false;
            if (ISO) {
                hit = iso_ray<COUNT>(A.S, A.iflags, A.M, r, tmin, tmax, rho, t_hit, g, st);
                if (hit) t_end = t_hit;
            }
            volume_ray<GRAD, COUNT>(A.S, A.vflags, A.M, s_tf, r, tmin, t_end, rho, acc, st);
            if (ISO && hit) {
                const double f = shade_factor(g, r);
                const double w = 1.0 - acc[3];
                acc[0] += w * A.M.iso_rgb[0] * f;
                acc[1] += w * A.M.iso_rgb[1] * f;
                acc[2] += w * A.M.iso_rgb[2] * f;
                acc[3] = 1.0;
            }
        }
        uchar4 q;
        unsigned char* qc = reinterpret_cast<unsigned char*>(&q);
#pragma unroll
        for (int c = 0; c < 4; c++) {
            double v = acc[c] < 0.0 ? 0.0 : acc[c];
            v = v > 1.0 ? 1.0 : v;
            qc[c] = (unsigned char)(v * 255.0 + 0.5);
        }
        const int64_t o = A.packed ? (int64_t)blockIdx.x * (kTileW * kTileH) + ly * kTileW + lx : pix;
        A.out8[o] = q;
        if (A.outf) A.outf[o] = make_double4(acc[0], acc[1], acc[2], acc[3]);
        if (A.outcnt) A.outcnt[o] = make_int2((int)st.regions, (int)st.samples);
    }
    // frame counters: warp reduce, then one atomic per warp into shared
    unsigned long long v0 = st.regions, v1 = st.samples, v2 = st.bytes;
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, o);
        v1 += __shfl_xor_sync(0xffffffffu, v1, o);
        v2 += __shfl_xor_sync(0xffffffffu, v2, o);
    }
    if (lane == 0) {
        atomicAdd(&s_stats[0], v0);
        atomicAdd(&s_stats[1], v1);
        if (COUNT) atomicAdd(&s_stats[2], v2);
    }
    __syncthreads();
    if (threadIdx.x == 0 && A.stats) {
        atomicAdd(&A.stats[0], s_stats[0]);
        atomicAdd(&A.stats[1], s_stats[1]);
        if (COUNT) atomicAdd(&A.stats[2], s_stats[2] + (unsigned long long)4 * kTileW * kTileH);
    }
}

using RenderFn = void (*)(RenderArgs);

template <int GRAD, bool ISO>
static RenderFn pick_count(bool count) {
    return count ? (RenderFn)k_render<GRAD, ISO, true> : (RenderFn)k_render<GRAD, ISO, false>;
}

template <int GRAD>
static RenderFn pick_iso(bool iso, bool count) {
    return iso ? pick_count<GRAD, true>(count) : pick_count<GRAD, false>(count);
}

void launch_render(const RenderArgs& A, int64_t n_tiles_local, bool count, cudaStream_t s) {
    if (n_tiles_local <= 0) return;
    RenderFn fn;
    const bool iso = A.M.iso_on != 0;
    switch (A.M.grad_mode) {
        case 0: fn = pick_iso<0>(iso, count); break;
        case 1: fn = pick_iso<1>(iso, count); break;
        default: fn = pick_iso<2>(iso, count); break;
    }
    void* args[] = {(void*)&A};
    XB_CUDA(cudaLaunchKernel((const void*)fn, dim3((unsigned)n_tiles_local), dim3(kTileW * kTileH), args, 0, s));
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
    if (B.mode == 0) {  // volume integration
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        clip_ray(B.M, r, tmin, tmax);
        if (tmin < tmax) {
            switch (B.M.grad_mode) {
                case 0: volume_ray<0, false>(B.S, B.vflags, B.M, s_tf, r, tmin, tmax, rho, acc, st); break;
                case 1: volume_ray<1, false>(B.S, B.vflags, B.M, s_tf, r, tmin, tmax, rho, acc, st); break;
                default: volume_ray<2, false>(B.S, B.vflags, B.M, s_tf, r, tmin, tmax, rho, acc, st); break;
            }
        }
        for (int c = 0; c < 4; c++) B.out[4 * q + c] = acc[c];
        B.counts[2 * q] = st.regions;
        B.counts[2 * q + 1] = st.samples;
    } else {  // iso intersection
        double g[3], th = 0.0;
        const bool hit = iso_ray<false>(B.S, B.iflags, B.M, r, tmin, tmax, rho, th, g, st);
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
