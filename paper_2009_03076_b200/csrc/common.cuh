// common.cuh — shared plumbing for libexabricks (sm_100a).
//
// Device data layout:
//   bricks   : int4  brick_a[B] = {lx, ly, lz, offset}      (16 B, one LDG.128)
//              u32   brick_m[B] = level | nx<<5 | ny<<14 | nz<<23
//   scalars  : f32   vals[F][N]  (x-fastest per brick, brick-major)
//   regions  : RegionRec[R] (32 B): half-unit box, brick-id range, finest level
//              i32   region_ids[]  (ascending brick ids per region)
//   k-d tree : KdNode[T] (8 B): BFS order, children adjacent; leaves carry the
//              region id (or -1 for a cavity outside the support union)
#pragma once
#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a profiler attached
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string>
#include <vector>
#include <stdexcept>
#include "../../include/exabricks.h"

namespace xb {

// ---------------------------------------------------------------------------
// errors: C++ exceptions inside the library, int status + thread-local text at
// the C ABI (include/exabricks.h).

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// status codes: XB_OK / XB_ERR_* from include/exabricks.h

#define XB_CUDA(call)                                                                          \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            char b_[512];                                                                      \
            snprintf(b_, sizeof b_, "%s failed at %s:%d: %s", #call, __FILE__, __LINE__,       \
                     cudaGetErrorString(e_));                                                  \
            throw ::xb::Error(XB_ERR_CUDA, b_);                                          \
        }                                                                                      \
    } while (0)

#define XB_CHECK(cond, code, msg)                                                              \
    do {                                                                                       \
        if (!(cond)) throw ::xb::Error((code), (msg));                                         \
    } while (0)

inline void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(XB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// device buffer (owning, move-only)

// Builder scratch (PoolScope): while a PoolScope is alive on this thread,
// DevBuf allocations come from a private per-device memory pool on the
// scope's stream.  The pool keeps what the builder frees (no release
// threshold), so the level-synchronous builders' grow-and-free cycles reuse
// mapped memory instead of cudaMalloc / cudaFree (each a device-wide
// synchronisation and a fresh mapping); the scope's end trims the pool back to
// what the built object still holds.  Buffers released inside the scope go
// back with cudaFreeAsync on its stream; buffers that outlive it (the built
// object) are released later with cudaFree, which accepts pool memory and
// waits for every stream using it.  Inside the scope every use of its buffers
// must be on its stream.
struct PoolCtx {
    cudaStream_t s = nullptr;
    cudaMemPool_t pool = nullptr;
};
inline PoolCtx& pool_scope() {
    thread_local PoolCtx c;
    return c;
}
cudaMemPool_t build_pool(int device);  // abi.cu
struct PoolScope {
    PoolCtx prev;
    explicit PoolScope(cudaStream_t s, int device) : prev(pool_scope()) { pool_scope() = PoolCtx{s, build_pool(device)}; }
    ~PoolScope() {
        const PoolCtx c = pool_scope();
        pool_scope() = prev;
        if (c.pool && cudaStreamSynchronize(c.s) == cudaSuccess) cudaMemPoolTrimTo(c.pool, 0);
    }
    PoolScope(const PoolScope&) = delete;
    PoolScope& operator=(const PoolScope&) = delete;
};

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    cudaStream_t ps = nullptr;  // stream of a pool allocation (PoolScope / alloc_async), else cudaMalloc'd
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), ps(o.ps) { o.p = nullptr; o.n = 0; o.ps = nullptr; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) { release(); p = o.p; n = o.n; ps = o.ps; o.p = nullptr; o.n = 0; o.ps = nullptr; }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        n = count;
        if (!count) return;
        const PoolCtx& c = pool_scope();
        if (c.pool) {
            XB_CUDA(cudaMallocFromPoolAsync((void**)&p, count * sizeof(T), c.pool, c.s));
            ps = c.s;
        } else {
            XB_CUDA(cudaMalloc(&p, count * sizeof(T)));
        }
    }
    // from the device's memory pool, ordered on stream s (no implicit device
    // synchronisation, retained pool memory: the TF-edit path); release() is
    // cudaFree, which accepts pool memory and waits for every stream using it
    void alloc_async(size_t count, cudaStream_t s) {
        release();
        n = count;
        if (count) XB_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), s));
        ps = count ? s : nullptr;
    }
    void ensure(size_t count) {  // grow-only
        if (count > n) alloc(count + count / 4 + 64);
    }
    void release() {
        if (p) {
            if (ps && ps == pool_scope().s) cudaFreeAsync(p, ps);  // scratch, still in its scope
            else cudaFree(p);
        }
        p = nullptr;
        n = 0;
        ps = nullptr;
    }
    void upload(const T* h, size_t count, cudaStream_t s = 0) {  // h: host or device (UVA)
        if (count > n) alloc(count);
        if (count) XB_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyDefault, s));
    }
    void download(T* h, size_t count, cudaStream_t s = 0) const {
        if (count) XB_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    std::vector<T> to_host(size_t count, cudaStream_t s = 0) const {
        std::vector<T> v(count);
        download(v.data(), count, s);
        XB_CUDA(cudaStreamSynchronize(s));
        return v;
    }
};

// stream-ordered scratch from the device's memory pool (cudaMallocAsync):
// no implicit device synchronisation on allocation or release, unlike
// cudaMalloc / cudaFree — a TF edit or a build never waits for other streams'
// renders
template <class T>
struct PoolBuf {
    T* p = nullptr;
    cudaStream_t s;
    PoolBuf(size_t count, cudaStream_t st) : s(st) {
        if (count) XB_CUDA(cudaMallocAsync((void**)&p, count * sizeof(T), s));
    }
    PoolBuf(const PoolBuf&) = delete;
    PoolBuf& operator=(const PoolBuf&) = delete;
    ~PoolBuf() {
        if (p) cudaFreeAsync(p, s);
    }
};

template <class T>
inline T read_scalar(const T* dptr, cudaStream_t s) {
    T v;
    XB_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    XB_CUDA(cudaStreamSynchronize(s));
    return v;
}

// RAII device guard: run on the object's device, restore the caller's
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        XB_CUDA(cudaGetDevice(&prev));
        if (prev != dev) XB_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        int cur;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

inline int grid_for(int64_t n, int block) { return (int)((n + block - 1) / block); }

// ---------------------------------------------------------------------------
// packed records

struct __align__(16) RegionRec {
    int32_t lo[3];      // half-unit box (world = value * 0.5, exact)
    int32_t hi[3];
    int32_t ids_begin;  // into region_ids
    int32_t meta;       // n_ids (low 24 bits) | finest level << 24
};
static_assert(sizeof(RegionRec) == 32, "RegionRec must be 32 bytes");

struct __align__(8) KdNode {
    int32_t a;  // interior: (left_child << 2) | axis ; leaf: -1 (cavity) or (region << 2) | 3
    int32_t b;  // interior: split plane in half units ; leaf: unused
};

// Two binary k-d levels collapsed into one 32-byte node (the warp traversal's
// node, csrc/kd4.cu).  Slots 0..3 are the grandchildren LL, LR, RL, RR (left =
// below the split plane); when a child of the root split is itself terminal
// its slot pair holds {child, -1}.  Child codes: >= 0 Kd4 node, -1 empty
// (cavity / unused), <= -2 leaf region -2 - code.
struct __align__(16) Kd4Node {
    int32_t plane[3];  // half units: [0] node split, [1] left child's split, [2] right child's split
    uint32_t axes;     // bits 0-1 axis of [0]; 2-3 / 4-5 axis of [1] / [2], 3 = child is terminal
    int32_t child[4];
};
static_assert(sizeof(Kd4Node) == 32, "Kd4Node must be 32 bytes");

__host__ __device__ inline uint32_t pack_brick_meta(int level, int nx, int ny, int nz) {
    return (uint32_t)level | ((uint32_t)nx << 5) | ((uint32_t)ny << 14) | ((uint32_t)nz << 23);
}

constexpr int kMaxDim = 511;       // per-axis brick width the packed meta can hold
constexpr int kMaxLevel = 30;

// ---------------------------------------------------------------------------
// device-resident model / regions / active sets (owned by ABI handles)

struct DevModel {
    int device = 0;
    int64_t n_bricks = 0, n_cells = 0;
    int n_fields = 0;
    int32_t coord_min = 0, coord_max = 0;     // bounds of brick boxes (for range checks)
    int max_level = 0;
    DevBuf<int4> brick_a;                     // {lx, ly, lz, offset}
    DevBuf<uint32_t> brick_m;                 // packed level/dims
    DevBuf<float> vals;                       // [F][N]
    // raw reference-layout arrays kept for download / region build
    DevBuf<int32_t> lower, level, dims;       // (B,3) (B) (B,3)
    DevBuf<int64_t> offset;                   // B+1
    // split tree of the brick build (SplitTree, R/bricks.py:45-68), preorder
    int64_t n_tree = 0;
    DevBuf<int32_t> t_axis, t_left, t_right, t_bstart, t_bcount;
    DevBuf<double> t_pos, t_lo, t_hi, t_mh;
};

struct DevRegions {
    int device = 0;
    int64_t n_regions = 0, n_ids = 0;
    int n_fields = 0;
    DevBuf<RegionRec> rec;
    DevBuf<int32_t> ids;
    DevBuf<float2> vrange;                    // [R][F] (min, max) — exact f32 values
    // k-d tree over the regions (the ABR build recursion), BFS order
    int64_t n_kd = 0;
    int kd_depth = 0;
    std::vector<int64_t> kd_level_base;       // BFS level boundaries (L+1 entries)
    int32_t root_lo[3] = {0, 0, 0}, root_hi[3] = {0, 0, 0};
    DevBuf<KdNode> kd;
    // the same tree with two levels per node (warp traversal), and the binary
    // node each slot stands for (to fold active flags into slot masks)
    int64_t n_kd4 = 0;
    DevBuf<Kd4Node> kd4;
    DevBuf<int4> kd4_bin;
    bool has_tree = false;
    // reference-layout arrays for download
    DevBuf<double> lo, hi, finest, vr64;
    DevBuf<int64_t> brick_off;
};

// host-side NVTX range for the phases of a call (visible in nsys / ncu --nvtx)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace xb
