// render.cu — the fused sm_100a ray-march kernels (paper §4-5) and the
// single-ray batch kernel behind integrate_ray / iso_intersect.
//
// k_frame (default): persistent warps.  Rays of one frame are "slots" in
// screen-tile order (16x8 tiles, 8x4 per warp chunk); a warp grabs 32 slots at
// a time from a global counter and every lane whose ray finished takes the
// next slot at once, so lanes stay busy although rays differ ~10x in length
// (visits per ray p50 36 / p99 186).  Each loop iteration a lane
// (1) finishes its region and fetches the next one from the ordered k-d walk,
// (2) refills with a new ray if its ray ended, (3) takes exactly one sample,
// so the expensive gather runs with (nearly) all lanes converged.
//
// k_render: one thread per pixel, one block per tile — kept as the simple
// reference kernel (XB_KERNEL=tile) for A/B measurements.
//
// The per-pixel arithmetic is `_render_kernel` (R/render.py:521-578) in both.
#include <cstdlib>
#include <cstring>
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
            if (iso_ray<COUNT>(A.S, A.iflags, A.M, r, tmin, tmax, rho, th, g, st)) {
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
// persistent frame kernel

struct LaneState {
    Ray r;
    KdWalk w;
    double rho, tmax;
    double acc[4];
    // current region
    const int32_t* ids;
    int nids, rid;
    double dt, s1, t_out, prev, k;
    // next region (found by the pipelined walk), query start of the walk
    int nrid;
    double nci, nco, q_t;
    int64_t slot, out;
    int nreg, nsmp;
};

enum : int { kSearching = 0, kFound = 1, kExhausted = 2 };

template <int GRAD, bool ISO, bool COUNT, int KSTEPS = kKdSteps, int MINB = kFrameMinBlocks>
__global__ void __launch_bounds__(kFrameThreads, MINB) k_frame(const __grid_constant__ RenderArgs A, int64_t n_slots) {
    __shared__ double s_tf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s_tf[i] = A.tf[i];
    __syncthreads();
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;

    LaneState L;
    bool has_ray = false, in_region = false, early = false;
    int nstate = kExhausted;
    int64_t chunk_next = 0, chunk_left = 0;
    bool exhausted = false;
    unsigned long long tot_reg = 0, tot_smp = 0, tot_bytes = 0;
    Accum G;

    for (;;) {
        // ---- prefetch the k-d node the walk visits this iteration (its latency
        //      hides behind the sample's gather)
        KdNode nd = {0, 0};
        uint8_t fl = 0;
        bool pre = has_ray && nstate == kSearching && L.w.node >= 0;  // cleared when the lane gets a new ray
        if (pre) {
            nd = A.S.kd[L.w.node];
            fl = A.vflags[L.w.node];
        }
        // ---- (1) promote the prefetched next region / finish the ray
        if (has_ray && !in_region) {
            if (!early && nstate == kFound) {
                const RegionRec rr = A.S.rec[L.nrid];
                L.rid = L.nrid;
                L.nids = rr.meta & 0xffffff;
                L.ids = A.S.rids + rr.ids_begin;
                const double fw = pow2(rr.meta >> 24);
                L.dt = fw / (A.M.spc * A.M.rate);
                L.s1 = fw / A.M.spc;
                L.t_out = L.nco;
                L.prev = L.nci;
                L.k = floor(L.nci / L.dt - L.rho) + 1.0;
                L.nreg++;
                if (COUNT) tot_bytes += 32 + 4 * (unsigned long long)L.nids;
                in_region = true;
                // the reference's next query: t = restart(t_out); stop if t >= tmax
                L.q_t = restart_t(L.nco);
                nstate = L.q_t >= L.tmax ? kExhausted : kSearching;
            } else if (early || nstate == kExhausted) {
                if (ISO) {
                    const double f = A.iso_shade[L.slot];
                    if (f >= 0.0) {
                        const double wgt = 1.0 - L.acc[3];
                        L.acc[0] += wgt * A.M.iso_rgb[0] * f;
                        L.acc[1] += wgt * A.M.iso_rgb[1] * f;
                        L.acc[2] += wgt * A.M.iso_rgb[2] * f;
                        L.acc[3] = 1.0;
                    }
                }
                write_pixel(A, L.out, L.acc, L.nreg, L.nsmp);
                tot_reg += L.nreg;
                tot_smp += L.nsmp;
                has_ray = false;
            }
        }
        // ---- (2) refill: lanes without a ray take the next slots of the warp's chunk
        bool want = !has_ray;
        unsigned need = __ballot_sync(FULL, want && !exhausted);
        while (need) {
            if (chunk_left == 0) {
                unsigned long long b = 0;
                if (lane == 0) b = atomicAdd(A.work_counter, 32ull);
                b = __shfl_sync(FULL, b, 0);
                chunk_next = (int64_t)b;
                chunk_left = (int64_t)b < n_slots ? min((int64_t)32, n_slots - (int64_t)b) : 0;
                if (chunk_left == 0) { exhausted = true; break; }
            }
            const int rank = __popc(need & lt_mask);
            const bool mine = want && rank < chunk_left;
            const int took = min(__popc(need), (int)chunk_left);
            const int64_t slot = chunk_next + rank;
            chunk_next += took;
            chunk_left -= took;
            if (mine) {
                const SlotPix sp = slot_pixel(A, slot);
                if (sp.live) {
                    pixel_ray(A, sp.x, sp.y, L.r);
                    L.rho = rho_hash((uint64_t)sp.pix, A.M.seed);
                    double tmin = 0.0, tmax = kTFar;
                    clip_ray(A.M, L.r, tmin, tmax);
                    L.slot = slot;
                    L.out = sp.out;
                    L.acc[0] = L.acc[1] = L.acc[2] = L.acc[3] = 0.0;
                    L.nreg = 0;
                    L.nsmp = 0;
                    if (tmin >= tmax) {
                        write_pixel(A, sp.out, L.acc, 0, 0);
                    } else {
                        L.tmax = ISO ? A.iso_tend[slot] : tmax;
                        L.q_t = tmin;
                        kd_begin(A.S, L.r, L.w);
                        pre = false;  // the prefetched node belonged to the previous ray
                        has_ray = true;
                        in_region = false;
                        early = false;
                        nstate = kSearching;
                    }
                }
                want = !has_ray;
            }
            need = __ballot_sync(FULL, want && !exhausted);
        }
        if (!__any_sync(FULL, has_ray)) {
            if (exhausted) break;
            continue;
        }
        // ---- (3) one sample (midpoint of the next lattice interval, R/render.py:406-449)
        if (in_region) {
            double tk;
            bool last = false;
            for (;;) {
                tk = L.dt * (L.k + L.rho);
                L.k += 1.0;
                if (tk >= L.t_out) { tk = L.t_out; last = true; break; }
                if (tk > L.prev) break;
            }
            const double sl = tk - L.prev;
            const double mid = 0.5 * (L.prev + tk);
            L.prev = tk;
            L.nsmp++;
            const double px = L.r.o[0] + mid * L.r.d[0], py = L.r.o[1] + mid * L.r.d[1], pz = L.r.o[2] + mid * L.r.d[2];
            gather_fast<GRAD == 1>(A.S, L.ids, L.nids, px, py, pz, G);
            if (COUNT) tot_bytes += 16 * (unsigned long long)L.nids + 4 * (unsigned long long)G.n_nz;
            if (G.den > kEpsWeight) {
                const double v = G.num / G.den;
                double c[4];
                tf_eval(s_tf, A.M.tf_lo, A.M.tf_hi, v, c);
                if (c[3] > 0.0) {
                    const double alpha = 1.0 - pow(1.0 - c[3], sl / L.s1);
                    if (GRAD != 0) {
                        double g[3];
                        if (GRAD == 1) {
                            analytic_gradient(G, g);
                        } else {
                            int64_t ne = 0;
                            central_gradient(A.S, A.M.grad_mode, px, py, pz, L.rid, L.ids, L.nids, v, g, &ne);
                        }
                        const double f = shade_factor(g, L.r);
                        c[0] *= f; c[1] *= f; c[2] *= f;
                    }
                    const double wgt = alpha * (1.0 - L.acc[3]);
                    L.acc[0] += wgt * c[0];
                    L.acc[1] += wgt * c[1];
                    L.acc[2] += wgt * c[2];
                    L.acc[3] += wgt;
                    if (L.acc[3] >= A.M.early) { last = true; early = true; }
                }
            }
            if (last) in_region = false;
        }
        // ---- (4) walk toward the next region: KSTEPS node visits
        if (has_ray && !early && nstate == kSearching) {
#pragma unroll 1
            for (int step = 0; step < KSTEPS; step++) {
                KdNode n2 = nd;
                uint8_t f2 = fl;
                if (!(pre && step == 0) && L.w.node >= 0) {
                    n2 = A.S.kd[L.w.node];
                    f2 = A.vflags[L.w.node];
                }
                int rid = -1;
                double ci = 0.0, co = 0.0;
                const int st = kd_step(A.S, A.vflags, L.r, L.w, n2, f2, L.q_t, L.tmax, rid, ci, co);
                if (st == 1) {
                    nstate = kFound;
                    L.nrid = rid;
                    L.nci = ci;
                    L.nco = co;
                    break;
                }
                if (st == 2) {
                    nstate = kExhausted;
                    break;
                }
            }
        }
    }
    // frame counters: one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
        tot_reg += __shfl_xor_sync(FULL, tot_reg, o);
        tot_smp += __shfl_xor_sync(FULL, tot_smp, o);
        tot_bytes += __shfl_xor_sync(FULL, tot_bytes, o);
    }
    if (lane == 0 && A.stats) {
        atomicAdd(&A.stats[0], tot_reg);
        atomicAdd(&A.stats[1], tot_smp);
        if (COUNT) atomicAdd(&A.stats[2], tot_bytes);
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
            volume_ray<GRAD, COUNT>(A.S, A.vflags, A.M, s_tf, r, tmin, t_end, rho, acc, st);
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
static FrameFn frame_fn(bool count) {
    return count ? (FrameFn)k_frame<GRAD, ISO, true> : (FrameFn)k_frame<GRAD, ISO, false>;
}

// tuning variants of the analytic, non-iso kernel (XB_KSTEPS / XB_MINB), for sweeps
static FrameFn tuned_fn(int ksteps, int minb) {
#define XB_T(K, B) if (ksteps == K && minb == B) return (FrameFn)k_frame<1, false, false, K, B>;
    XB_T(2, 4) XB_T(3, 4) XB_T(4, 4) XB_T(5, 4) XB_T(6, 4) XB_T(8, 4)
#undef XB_T
    return nullptr;
}
template <int GRAD, bool ISO>
static RenderFn tile_fn(bool count) {
    return count ? (RenderFn)k_render<GRAD, ISO, true> : (RenderFn)k_render<GRAD, ISO, false>;
}

static int grad_index(int mode) { return mode == 0 ? 0 : (mode == 1 ? 1 : 2); }

static bool use_tile_kernel() {
    const char* e = getenv("XB_KERNEL");
    return e && strcmp(e, "tile") == 0;
}

void launch_render(const RenderArgs& A, int64_t n_tiles_local, bool count, cudaStream_t s) {
    if (n_tiles_local <= 0) return;
    const bool iso = A.M.iso_on != 0;
    const int g = grad_index(A.M.grad_mode);
    const int64_t n_slots = n_tiles_local * kTileW * kTileH;
    if (iso) {
        void* args[] = {(void*)&A, (void*)&n_slots};
        const void* fn = count ? (const void*)k_iso_pass<true> : (const void*)k_iso_pass<false>;
        XB_CUDA(cudaLaunchKernel(fn, dim3(grid_for(n_slots, 128)), dim3(128), args, 0, s));
    }
    if (use_tile_kernel()) {
        RenderFn fn;
        if (g == 0) fn = iso ? tile_fn<0, true>(count) : tile_fn<0, false>(count);
        else if (g == 1) fn = iso ? tile_fn<1, true>(count) : tile_fn<1, false>(count);
        else fn = iso ? tile_fn<2, true>(count) : tile_fn<2, false>(count);
        void* args[] = {(void*)&A};
        XB_CUDA(cudaLaunchKernel((const void*)fn, dim3((unsigned)n_tiles_local), dim3(kTileW * kTileH), args, 0, s));
        return;
    }
    FrameFn fn;
    if (g == 0) fn = iso ? frame_fn<0, true>(count) : frame_fn<0, false>(count);
    else if (g == 1) fn = iso ? frame_fn<1, true>(count) : frame_fn<1, false>(count);
    else fn = iso ? frame_fn<2, true>(count) : frame_fn<2, false>(count);
    if (g == 1 && !iso && !count && (getenv("XB_KSTEPS") || getenv("XB_MINB"))) {
        const int ks = getenv("XB_KSTEPS") ? atoi(getenv("XB_KSTEPS")) : kKdSteps;
        const int mb = getenv("XB_MINB") ? atoi(getenv("XB_MINB")) : 4;
        if (FrameFn t = tuned_fn(ks, mb)) fn = t;
    }
    int dev = 0, sms = 0, per_sm = 0;
    XB_CUDA(cudaGetDevice(&dev));
    XB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    XB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, kFrameThreads, 0));
    const int64_t want = (n_slots + kFrameThreads - 1) / kFrameThreads;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), want));
    void* args[] = {(void*)&A, (void*)&n_slots};
    XB_CUDA(cudaLaunchKernel((const void*)fn, dim3((unsigned)blocks), dim3(kFrameThreads), args, 0, s));
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
