// scan.cuh — CUB-backed device scans / sorts with cached temp storage.
#pragma once
#include <cub/cub.cuh>
#include "common.cuh"

namespace xb {

struct CubTemp {
    DevBuf<char> buf;
    void* get(size_t bytes) {
        buf.ensure(bytes ? bytes : 1);
        return buf.p;
    }
};

// CUB scratch from the stream's memory pool (see PoolBuf)
struct CubPoolTemp {
    cudaStream_t s;
    char* p = nullptr;
    size_t n = 0;
    explicit CubPoolTemp(cudaStream_t st) : s(st) {}
    CubPoolTemp(const CubPoolTemp&) = delete;
    CubPoolTemp& operator=(const CubPoolTemp&) = delete;
    void* get(size_t bytes) {
        if (bytes > n) {
            if (p) XB_CUDA(cudaFreeAsync(p, s));
            n = bytes ? bytes : 1;
            XB_CUDA(cudaMallocAsync((void**)&p, n, s));
        }
        return p;
    }
    ~CubPoolTemp() {
        if (p) cudaFreeAsync(p, s);
    }
};

// out[i] = sum(in[0..i)), n+1 outputs when `in` has n+1 entries with in[n] = 0
template <class T, class Tmp>
inline void exclusive_sum(Tmp& tmp, const T* in, T* out, int64_t n, cudaStream_t s) {
    size_t bytes = 0;
    XB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
    XB_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(bytes), bytes, in, out, n, s));
}

template <class K, class V>
inline void sort_pairs(CubTemp& tmp, const K* kin, K* kout, const V* vin, V* vout, int64_t n, int begin_bit, int end_bit,
                       cudaStream_t s) {
    size_t bytes = 0;
    XB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, begin_bit, end_bit, s));
    XB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(bytes), bytes, kin, kout, vin, vout, n, begin_bit, end_bit, s));
}

template <class T>
inline T reduce_max(CubTemp& tmp, const T* in, int64_t n, DevBuf<T>& out1, cudaStream_t s) {
    out1.ensure(1);
    size_t bytes = 0;
    XB_CUDA(cub::DeviceReduce::Max(nullptr, bytes, in, out1.p, n, s));
    XB_CUDA(cub::DeviceReduce::Max(tmp.get(bytes), bytes, in, out1.p, n, s));
    return read_scalar(out1.p, s);
}

template <class T>
inline T reduce_min(CubTemp& tmp, const T* in, int64_t n, DevBuf<T>& out1, cudaStream_t s) {
    out1.ensure(1);
    size_t bytes = 0;
    XB_CUDA(cub::DeviceReduce::Min(nullptr, bytes, in, out1.p, n, s));
    XB_CUDA(cub::DeviceReduce::Min(tmp.get(bytes), bytes, in, out1.p, n, s));
    return read_scalar(out1.p, s);
}

// grow a device buffer preserving contents
template <class T>
inline void grow_keep(DevBuf<T>& b, size_t need, size_t used, cudaStream_t s) {
    if (need <= b.n) return;
    DevBuf<T> nb(need + need / 2 + 1024);
    if (used) XB_CUDA(cudaMemcpyAsync(nb.p, b.p, used * sizeof(T), cudaMemcpyDeviceToDevice, s));
    XB_CUDA(cudaStreamSynchronize(s));
    b = std::move(nb);
}

// warp-aggregated atomics for segment-contiguous reductions: when every active
// lane of the warp targets the same node, reduce in registers first.
__device__ __forceinline__ bool warp_uniform(unsigned mask, int key) {
    int k0 = __shfl_sync(mask, key, __ffs(mask) - 1);
    return __all_sync(mask, key == k0);
}

}  // namespace xb
