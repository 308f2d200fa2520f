// abi.cu — extern "C" entry points of libexabricks (include/exabricks.h).
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <vector>
#include "../../include/exabricks.h"
#include "accel.cuh"
#include "render.cuh"
#include "synth.cuh"

namespace xb {
bool build_bricks_device(const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* l, const float* v,
                         int64_t n, int F, int64_t maxw, bool keep_tree, int device, DevModel& m, cudaStream_t s);
void finish_model(DevModel& m, cudaStream_t s);
void build_regions_device(const DevModel& m, DevRegions& out, cudaStream_t s);
}  // namespace xb

struct xb_cells {
    xb::DevCells c;
};
// the builders' private pool per device (common.cuh:PoolScope)
namespace xb {
cudaMemPool_t build_pool(int device) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    std::lock_guard<std::mutex> g(mu);
    XB_CHECK(device >= 0 && device < 64, XB_ERR_ARG, "device index out of range");
    if (!pools[device]) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = device;
        XB_CUDA(cudaMemPoolCreate(&pools[device], &props));
        uint64_t keep = UINT64_MAX;  // trimmed explicitly at each PoolScope's end
        XB_CUDA(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep));
    }
    return pools[device];
}
}  // namespace xb

struct xb_model {
    xb::DevModel m;
    // the frame gather's padded copy of each rendered field (march.cuh:kGatherPad), built
    // on the field's first render and kept for the model's life (concurrent renders
    // of other fields never see it move)
    mutable std::mutex gv_mu;
    mutable std::vector<std::unique_ptr<xb::DevBuf<float>>> gvals;
};
struct xb_regions {
    xb::DevRegions r;
    int64_t model_bricks = 0;
    // brick records in region-list order for the frame gather (built on first render)
    mutable std::mutex rb_mu;
    mutable xb::DevBuf<xb::RbRec> rb;
    mutable bool rb_ok = false;
};
struct xb_active {
    xb::DevActive a;
    const xb_regions* owner = nullptr;
};

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return XB_OK;
    } catch (const xb::Error& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return XB_ERR_INTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return XB_ERR_INTERNAL;
    }
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// per-call owned stream for synchronous builders
struct OwnedStream {
    cudaStream_t s = nullptr;
    OwnedStream() { XB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
    ~OwnedStream() {
        if (s) cudaStreamDestroy(s);
    }
};

// keep up to 8 GB of freed stream-ordered allocations in the device pool: a
// frame's scratch (<= ~4 GB, see kBandSlots) is reused every frame instead of
// going back to the driver, while larger or concurrent peaks are released at
// the next synchronisation instead of being held for the life of the process
void keep_pool(int device) {
    static std::once_flag done[64];
    if (device < 0 || device >= 64) return;
    std::call_once(done[device], [device] {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = 8ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    });
}

// pixels rendered per pass; larger frames run as interleaved tile bands (xb_render)
constexpr int64_t kBandSlots = 1ll << 22;

// frame-gather brick records in region-list order (march.cuh:RbRec)
__global__ void k_region_bricks(const int32_t* __restrict__ ids, int64_t n, const int4* __restrict__ ba,
                                const uint32_t* __restrict__ bm, xb::RbRec* __restrict__ rb) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int b = ids[i];
    const int4 a = ba[b];
    xb::RbRec r;
    r.lx = (double)a.x;
    r.ly = (double)a.y;
    r.lz = (double)a.z;
    r.off = (uint32_t)a.w;
    r.meta = bm[b];
    rb[i] = r;
}

void ensure_region_bricks(const xb_model* m, const xb_regions* r) {
    std::lock_guard<std::mutex> g(r->rb_mu);
    if (r->rb_ok) return;
    const int64_t n = std::max<int64_t>(r->r.n_ids, 1);
    r->rb.alloc(n);
    if (r->r.n_ids > 0) {
        OwnedStream st;
        k_region_bricks<<<(unsigned)((r->r.n_ids + 255) / 256), 256, 0, st.s>>>(
            r->r.ids.p, r->r.n_ids, m->m.brick_a.p, m->m.brick_m.p, r->rb.p);
        XB_CUDA(cudaGetLastError());
        XB_CUDA(cudaStreamSynchronize(st.s));
    }
    r->rb_ok = true;
}

// the field's values with kGatherPad zeros on both sides (march.cuh:brick_step)
const float* gather_values(const xb_model* m, int field) {
    std::lock_guard<std::mutex> g(m->gv_mu);
    if ((int)m->gvals.size() <= field) m->gvals.resize(field + 1);
    if (!m->gvals[field]) {
        const int64_t n = m->m.n_cells, pad = xb::kGatherPad;
        auto b = std::make_unique<xb::DevBuf<float>>((size_t)(n + 2 * pad));
        OwnedStream st;
        XB_CUDA(cudaMemsetAsync(b->p, 0, (size_t)(n + 2 * pad) * sizeof(float), st.s));
        if (n)
            XB_CUDA(cudaMemcpyAsync(b->p + pad, m->m.vals.p + (size_t)field * (size_t)n, (size_t)n * sizeof(float),
                                    cudaMemcpyDeviceToDevice, st.s));
        XB_CUDA(cudaStreamSynchronize(st.s));
        m->gvals[field] = std::move(b);
    }
    return m->gvals[field]->p + xb::kGatherPad;
}

xb::SceneView scene_view(const xb_model* m, const xb_regions* r, int field) {
    XB_CHECK(m && r, XB_ERR_ARG, "null model or regions");
    XB_CHECK(r->model_bricks == m->m.n_bricks, XB_ERR_ARG, "regions were built for a different model");
    XB_CHECK(field >= 0 && field < std::max(m->m.n_fields, 1), XB_ERR_ARG, "field index out of range");
    XB_CHECK(r->r.has_tree, XB_ERR_NO_TREE, "regions carry no k-d tree");
    XB_CHECK(r->r.kd_depth <= xb::kKdStack, XB_ERR_RANGE, "region k-d tree deeper than the traversal stack");
    xb::SceneView S;
    S.brick_a = m->m.brick_a.p;
    S.brick_m = m->m.brick_m.p;
    S.vals = m->m.vals.p + (size_t)field * (size_t)m->m.n_cells;
    S.gvals = gather_values(m, field);
    S.rec = r->r.rec.p;
    S.rids = r->r.ids.p;
    ensure_region_bricks(m, r);
    S.rb = r->rb.p;
    S.kd = r->r.kd.p;
    S.kd4 = r->r.kd4.p;
    for (int a = 0; a < 3; a++) {
        S.root_lo[a] = r->r.root_lo[a];
        S.root_hi[a] = r->r.root_hi[a];
    }
    S.n_kd = r->r.n_regions > 0 ? r->r.n_kd : 0;
    const xb::DevModel& d = m->m;
    S.tree = xb::TreeView{d.t_axis.p, d.t_left.p, d.t_right.p, d.t_bstart.p, d.t_bcount.p, d.t_lo.p, d.t_hi.p,
                          d.t_mh.p, d.n_tree};
    S.n_kd4 = r->r.n_regions > 0 ? r->r.n_kd4 : 0;
    return S;
}

void fill_march(xb::MarchConst& M, const xb_march* mp) {
    M.spc = mp->samples_per_cell;
    M.rate = mp->rate_scale;
    M.early = mp->early_term_threshold;
    M.seed = mp->seed;
    M.grad_mode = mp->gradient_mode;
    XB_CHECK(mp->gradient_mode >= 0 && mp->gradient_mode <= 3, XB_ERR_ARG, "unknown gradient mode");
    XB_CHECK(mp->n_planes >= 0 && mp->n_planes <= 6, XB_ERR_ARG, "at most 6 clip planes are supported");
    M.n_planes = mp->n_planes;
    for (int i = 0; i < 6; i++)
        for (int c = 0; c < 4; c++) M.planes[i][c] = mp->planes[i][c];
    M.iso_on = mp->iso_on;
    M.iso_value = mp->iso_value;
    for (int c = 0; c < 3; c++) M.iso_rgb[c] = mp->iso_rgb[c];
    M.tf_lo = mp->tf_lo;
    M.tf_hi = mp->tf_hi;
    M.tf_den = mp->tf_hi - mp->tf_lo;
    M.tf_inv = 1.0 / M.tf_den;
    M.use_tree = mp->use_tree;
    for (int l = 0; l < 32; l++) {
        const double fw = std::ldexp(1.0, l);
        M.lv_dt[l] = fw / (M.spc * M.rate);
        M.lv_s1[l] = fw / M.spc;
        M.lv_is1[l] = 1.0 / M.lv_s1[l];
        int ex = 0;
        M.lv_idt[l] = std::frexp(M.lv_dt[l], &ex) == 0.5 ? std::ldexp(1.0, 1 - ex) : 0.0;  // dt = 2^(ex-1)
    }
}

void check_active(const xb_active* a, const xb_regions* r, const char* what) {
    XB_CHECK(a != nullptr, XB_ERR_ARG, std::string(what) + " active set is NULL");
    XB_CHECK(a->owner == r, XB_ERR_ARG, std::string(what) + " active set belongs to other regions");
}

// device staging for an optional host/device output
template <class T>
struct OutBuf {
    T* user = nullptr;
    T* dev = nullptr;
    size_t count = 0;
    bool owned = false;
    cudaStream_t s = nullptr;
    void setup(T* p, size_t n, cudaStream_t st) {
        user = p;
        count = n;
        s = st;
        if (!p) return;
        if (is_device_ptr(p)) {
            dev = p;
        } else {
            XB_CUDA(cudaMallocAsync((void**)&dev, std::max<size_t>(n, 1) * sizeof(T), s));
            owned = true;
        }
    }
    void finish() {
        if (owned && count) XB_CUDA(cudaMemcpyAsync(user, dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    }
    ~OutBuf() {
        if (owned && dev) cudaFreeAsync(dev, s);
    }
};

int64_t tiles_for_rank(int W, int H, int rank, int world, int* tx_o, int* ty_o) {
    const int tx = (W + xb::kTileW - 1) / xb::kTileW, ty = (H + xb::kTileH - 1) / xb::kTileH;
    if (tx_o) *tx_o = tx;
    if (ty_o) *ty_o = ty;
    const int64_t total = (int64_t)tx * ty;
    if (rank >= total) return 0;
    return (total - rank + world - 1) / world;
}

}  // namespace

extern "C" {

const char* xb_last_error(void) { return g_err.c_str(); }

int xb_abi_version(void) { return 1; }

int xb_device_count(int32_t* n) {
    return guarded([&] {
        int c = 0;
        XB_CUDA(cudaGetDeviceCount(&c));
        *n = c;
    });
}

int xb_build_bricks(const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* level, const float* values,
                    int64_t n, int32_t n_fields, int32_t max_brick_width, int32_t keep_split_tree, int32_t device,
                    xb_model** out) {
    *out = nullptr;
    return guarded([&] {
        xb::NvtxRange nvtx_range("xb_build_bricks");
        XB_CHECK(n >= 0 && n_fields >= 1, XB_ERR_ARG, "bad cell counts");
        xb::DeviceGuard g(device);
        OwnedStream st;
        auto h = std::make_unique<xb_model>();
        bool ok = xb::build_bricks_device(i, j, k, level, values, n, n_fields, max_brick_width, keep_split_tree != 0,
                                          device, h->m, st.s);
        XB_CHECK(ok, XB_ERR_INVALID_CELLS, "cells fail validation (alignment, duplicates or overlaps)");
        *out = h.release();
    });
}

int xb_generate_synthetic(const xb_synth_spec* spec, int32_t device, xb_cells** out) {
    *out = nullptr;
    return guarded([&] {
        xb::NvtxRange nvtx_range("xb_generate_synthetic");
        XB_CHECK(spec != nullptr, XB_ERR_ARG, "null spec");
        xb::DeviceGuard g(device);
        OwnedStream st;
        auto h = std::make_unique<xb_cells>();
        xb::generate_synthetic_device(*spec, device, h->c, st.s);
        *out = h.release();
    });
}

int xb_cells_info(const xb_cells* c, int64_t* n) {
    return guarded([&] {
        XB_CHECK(c && n, XB_ERR_ARG, "null argument");
        *n = c->c.n;
    });
}

int xb_cells_download(const xb_cells* c, int32_t* i, int32_t* j, int32_t* k, int32_t* level, float* values) {
    return guarded([&] {
        XB_CHECK(c != nullptr, XB_ERR_ARG, "null cells");
        xb::DeviceGuard g(c->c.device);
        OwnedStream st;
        const size_t n = (size_t)c->c.n;
        if (i) c->c.i.download(i, n, st.s);
        if (j) c->c.j.download(j, n, st.s);
        if (k) c->c.k.download(k, n, st.s);
        if (level) c->c.level.download(level, n, st.s);
        if (values) c->c.vals.download(values, n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

void xb_cells_free(xb_cells* c) { delete c; }

int xb_cells_create(int64_t n, int32_t device, xb_cells** out) {
    *out = nullptr;
    return guarded([&] {
        XB_CHECK(n >= 0 && n < (1ll << 31) - 2, XB_ERR_RANGE, "cell count out of range");
        xb::DeviceGuard g(device);
        auto h = std::make_unique<xb_cells>();
        h->c.device = device;
        h->c.n = n;
        h->c.i.alloc(n + 1); h->c.j.alloc(n + 1); h->c.k.alloc(n + 1); h->c.level.alloc(n + 1);
        h->c.vals.alloc(n + 1);
        *out = h.release();
    });
}

int xb_cells_upload(xb_cells* c, int64_t offset, int64_t count, const int32_t* i, const int32_t* j, const int32_t* k,
                    const int32_t* level, const float* values) {
    return guarded([&] {
        XB_CHECK(c && offset >= 0 && count >= 0 && offset + count <= c->c.n, XB_ERR_ARG, "upload range out of bounds");
        xb::DeviceGuard g(c->c.device);
        OwnedStream st;
        const size_t b4 = (size_t)count * 4;
        if (count) {
            XB_CUDA(cudaMemcpyAsync(c->c.i.p + offset, i, b4, cudaMemcpyDefault, st.s));
            XB_CUDA(cudaMemcpyAsync(c->c.j.p + offset, j, b4, cudaMemcpyDefault, st.s));
            XB_CUDA(cudaMemcpyAsync(c->c.k.p + offset, k, b4, cudaMemcpyDefault, st.s));
            XB_CUDA(cudaMemcpyAsync(c->c.level.p + offset, level, b4, cudaMemcpyDefault, st.s));
            XB_CUDA(cudaMemcpyAsync(c->c.vals.p + offset, values, b4, cudaMemcpyDefault, st.s));
        }
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_build_bricks_cells(const xb_cells* c, int32_t max_brick_width, int32_t keep_split_tree, xb_model** out) {
    *out = nullptr;
    return guarded([&] {
        xb::NvtxRange nvtx_range("xb_build_bricks (device cells)");
        XB_CHECK(c != nullptr, XB_ERR_ARG, "null cells");
        xb::DeviceGuard g(c->c.device);
        OwnedStream st;
        auto h = std::make_unique<xb_model>();
        bool ok = xb::build_bricks_device(c->c.i.p, c->c.j.p, c->c.k.p, c->c.level.p, c->c.vals.p, c->c.n, 1,
                                          max_brick_width, keep_split_tree != 0, c->c.device, h->m, st.s);
        XB_CHECK(ok, XB_ERR_INVALID_CELLS, "cells fail validation (alignment, duplicates or overlaps)");
        *out = h.release();
    });
}

int xb_model_upload(const int32_t* lower, const int32_t* level, const int32_t* dims, const float* scalars,
                    int64_t n_bricks, int64_t n_cells, int32_t n_fields, int32_t device, xb_model** out) {
    *out = nullptr;
    return guarded([&] {
        XB_CHECK(n_bricks >= 0 && n_cells >= 0 && n_fields >= 1, XB_ERR_ARG, "bad model sizes");
        xb::DeviceGuard g(device);
        OwnedStream st;
        auto h = std::make_unique<xb_model>();
        xb::DevModel& m = h->m;
        m.device = device;
        m.n_bricks = n_bricks;
        m.n_fields = n_fields;
        std::vector<int64_t> off(n_bricks + 1, 0);
        for (int64_t b = 0; b < n_bricks; b++)
            off[b + 1] = off[b] + (int64_t)dims[3 * b] * dims[3 * b + 1] * dims[3 * b + 2];
        XB_CHECK(off[n_bricks] == n_cells, XB_ERR_ARG, "scalar array length does not match brick dims");
        m.n_cells = n_cells;
        m.lower.upload(lower, 3 * n_bricks, st.s);
        m.level.upload(level, n_bricks, st.s);
        m.dims.upload(dims, 3 * n_bricks, st.s);
        m.offset.upload(off.data(), n_bricks + 1, st.s);
        m.vals.alloc((size_t)n_fields * n_cells + 1);
        if (n_cells) XB_CUDA(cudaMemcpyAsync(m.vals.p, scalars, (size_t)n_fields * n_cells * 4, cudaMemcpyHostToDevice, st.s));
        xb::finish_model(m, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
        *out = h.release();
    });
}

int xb_model_upload_tree(xb_model* m, int64_t n, const int32_t* axis, const double* pos, const int32_t* left,
                         const int32_t* right, const int32_t* brick_start, const int32_t* brick_count,
                         const double* box_lo, const double* box_hi, const double* max_half) {
    return guarded([&] {
        XB_CHECK(m && n >= 0, XB_ERR_ARG, "bad tree upload");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        xb::DevModel& d = m->m;
        d.n_tree = n;
        d.t_axis.upload(axis, n, st.s);
        d.t_pos.upload(pos, n, st.s);
        d.t_left.upload(left, n, st.s);
        d.t_right.upload(right, n, st.s);
        d.t_bstart.upload(brick_start, n, st.s);
        d.t_bcount.upload(brick_count, n, st.s);
        d.t_lo.upload(box_lo, 3 * n, st.s);
        d.t_hi.upload(box_hi, 3 * n, st.s);
        d.t_mh.upload(max_half, n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_model_info(const xb_model* m, int64_t* n_bricks, int64_t* n_cells, int32_t* n_fields, int64_t* n_tree_nodes) {
    return guarded([&] {
        XB_CHECK(m, XB_ERR_ARG, "null model");
        if (n_bricks) *n_bricks = m->m.n_bricks;
        if (n_cells) *n_cells = m->m.n_cells;
        if (n_fields) *n_fields = m->m.n_fields;
        if (n_tree_nodes) *n_tree_nodes = m->m.n_tree;
    });
}

int xb_model_download(const xb_model* m, int32_t* lower, int32_t* level, int32_t* dims, int64_t* offset,
                      float* scalars) {
    return guarded([&] {
        XB_CHECK(m, XB_ERR_ARG, "null model");
        xb::DeviceGuard g(m->m.device);
        const auto& d = m->m;
        const int64_t B = d.n_bricks;
        if (lower) d.lower.download(lower, 3 * B);
        if (level) d.level.download(level, B);
        if (dims) d.dims.download(dims, 3 * B);
        if (offset) d.offset.download(offset, B + 1);
        if (scalars) d.vals.download(scalars, (size_t)d.n_fields * d.n_cells);
        XB_CUDA(cudaStreamSynchronize(0));
    });
}

int xb_model_download_tree(const xb_model* m, int32_t* axis, double* pos, int32_t* left, int32_t* right,
                           int32_t* brick_start, int32_t* brick_count, double* box_lo, double* box_hi,
                           double* max_half) {
    return guarded([&] {
        XB_CHECK(m, XB_ERR_ARG, "null model");
        xb::DeviceGuard g(m->m.device);
        const auto& d = m->m;
        const int64_t T = d.n_tree;
        d.t_axis.download(axis, T);
        d.t_pos.download(pos, T);
        d.t_left.download(left, T);
        d.t_right.download(right, T);
        d.t_bstart.download(brick_start, T);
        d.t_bcount.download(brick_count, T);
        d.t_lo.download(box_lo, 3 * T);
        d.t_hi.download(box_hi, 3 * T);
        d.t_mh.download(max_half, T);
        XB_CUDA(cudaStreamSynchronize(0));
    });
}

void xb_model_free(xb_model* m) {
    if (!m) return;
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(m->m.device);
    delete m;
    cudaSetDevice(prev);
}

int xb_build_regions(const xb_model* m, xb_regions** out) {
    *out = nullptr;
    return guarded([&] {
        xb::NvtxRange nvtx_range("xb_build_regions");
        XB_CHECK(m, XB_ERR_ARG, "null model");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        // scratch from the builders' pool (common.cuh:PoolScope): C3 regions 0.32-0.99 s
        // over 8 rebuilds against 0.58-1.5 s through cudaMalloc (build_bricks, whose
        // 30 GB peak maps faster as a few cudaMalloc blocks, keeps cudaMalloc)
        xb::PoolScope pool(st.s, m->m.device);
        auto h = std::make_unique<xb_regions>();
        xb::build_regions_device(m->m, h->r, st.s);
        h->model_bricks = m->m.n_bricks;
        *out = h.release();
    });
}

int xb_regions_info(const xb_regions* r, int64_t* n_regions, int64_t* n_ids, int64_t* n_kd_nodes, int32_t* kd_depth) {
    return guarded([&] {
        XB_CHECK(r, XB_ERR_ARG, "null regions");
        if (n_regions) *n_regions = r->r.n_regions;
        if (n_ids) *n_ids = r->r.n_ids;
        if (n_kd_nodes) *n_kd_nodes = r->r.n_kd;
        if (kd_depth) *kd_depth = r->r.kd_depth;
    });
}

int xb_regions_download(const xb_regions* r, double* lo, double* hi, int64_t* brick_off, int32_t* brick_ids,
                        double* value_range, double* finest_width) {
    return guarded([&] {
        XB_CHECK(r, XB_ERR_ARG, "null regions");
        xb::DeviceGuard g(r->r.device);
        const auto& d = r->r;
        const int64_t R = d.n_regions;
        if (lo) d.lo.download(lo, 3 * R);
        if (hi) d.hi.download(hi, 3 * R);
        if (brick_off) d.brick_off.download(brick_off, R + 1);
        if (brick_ids) d.ids.download(brick_ids, d.n_ids);
        if (value_range) d.vr64.download(value_range, 2 * R * d.n_fields);
        if (finest_width) d.finest.download(finest_width, R);
        XB_CUDA(cudaStreamSynchronize(0));
    });
}

void xb_regions_free(xb_regions* r) {
    if (!r) return;
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(r->r.device);
    delete r;
    cudaSetDevice(prev);
}

static int make_active(const xb_regions* r, int kind, int32_t field, double lo, double hi, const double* rgba,
                       double iso, xb_active** out) {
    *out = nullptr;
    return guarded([&] {
        xb::NvtxRange nvtx_range(kind == 0 ? "active set: volume majorants" : (kind == 1 ? "active set: iso" : "active set: all"));
        XB_CHECK(r, XB_ERR_ARG, "null regions");
        if (kind == 0) XB_CHECK(rgba && lo < hi, XB_ERR_ARG, "transfer function domain must satisfy lo < hi");
        xb::DeviceGuard g(r->r.device);
        OwnedStream st;
        auto h = std::make_unique<xb_active>();
        auto t0 = std::chrono::steady_clock::now();
        xb::build_active(r->r, kind, field, lo, hi, rgba, iso, h->a, st.s);
        h->a.build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        h->owner = r;
        *out = h.release();
    });
}

int xb_active_volume(const xb_regions* r, int32_t field, double tf_lo, double tf_hi, const double* rgba,
                     xb_active** out) {
    return make_active(r, 0, field, tf_lo, tf_hi, rgba, 0.0, out);
}

int xb_active_iso(const xb_regions* r, int32_t field, double iso_value, xb_active** out) {
    return make_active(r, 1, field, 0.0, 1.0, nullptr, iso_value, out);
}

int xb_active_all(const xb_regions* r, xb_active** out) { return make_active(r, 2, 0, 0.0, 1.0, nullptr, 0.0, out); }

int xb_active_info(const xb_active* a, int64_t* n_active, double* build_ms) {
    return guarded([&] {
        XB_CHECK(a, XB_ERR_ARG, "null active set");
        if (n_active) *n_active = a->a.n_active;
        if (build_ms) *build_ms = a->a.build_ms;
    });
}

int xb_active_prims(const xb_active* a, int32_t* prims) {
    return guarded([&] {
        XB_CHECK(a, XB_ERR_ARG, "null active set");
        xb::DeviceGuard g(a->a.device);
        a->a.prims.download(prims, a->a.n_active);
        XB_CUDA(cudaStreamSynchronize(0));
    });
}

void xb_active_free(xb_active* a) {
    if (!a) return;
    int prev;
    cudaGetDevice(&prev);
    cudaSetDevice(a->a.device);
    delete a;
    cudaSetDevice(prev);
}

int xb_tile_count(int32_t width, int32_t height, int32_t rank, int32_t world, int64_t* n_tiles, int32_t* tile_px) {
    return guarded([&] {
        XB_CHECK(width >= 1 && height >= 1 && world >= 1 && rank >= 0 && rank < world, XB_ERR_ARG, "bad tiling");
        if (n_tiles) *n_tiles = tiles_for_rank(width, height, rank, world, nullptr, nullptr);
        if (tile_px) *tile_px = xb::kTileW * xb::kTileH;
    });
}

namespace {
std::mutex g_tuning_mu;
xb_tuning g_tuning = [] {
    xb_tuning t;
    xb_tuning_defaults(&t);
    return t;
}();

xb_tuning tuning_snapshot() {
    std::lock_guard<std::mutex> g(g_tuning_mu);
    return g_tuning;
}

// k_warp event pairs of frames rendered with tuning.time_march (xb_march_times)
struct MarchEvents {
    int device;
    cudaEvent_t ev[2];
};
std::mutex g_events_mu;
std::vector<MarchEvents> g_events;
}  // namespace

int xb_march_times(double* ms, int32_t cap, int32_t* n) {
    return guarded([&] {
        XB_CHECK(n && (ms || cap == 0) && cap >= 0, XB_ERR_ARG, "bad march-times arguments");
        std::vector<MarchEvents> take;
        {
            std::lock_guard<std::mutex> g(g_events_mu);
            const size_t k = std::min<size_t>(g_events.size(), (size_t)cap);
            take.assign(g_events.begin(), g_events.begin() + k);
            g_events.erase(g_events.begin(), g_events.begin() + k);
        }
        int32_t got = 0;
        for (auto& e : take) {
            xb::DeviceGuard dg(e.device);
            float t = 0.f;
            XB_CUDA(cudaEventSynchronize(e.ev[1]));
            XB_CUDA(cudaEventElapsedTime(&t, e.ev[0], e.ev[1]));
            ms[got++] = (double)t;
            cudaEventDestroy(e.ev[0]);
            cudaEventDestroy(e.ev[1]);
        }
        *n = got;
    });
}

void xb_tuning_defaults(xb_tuning* t) {
    if (!t) return;
    std::memset(t, 0, sizeof(*t));
    t->kernel = 0;
    t->traversal = 0;
    t->walk_lists = 1;
    t->leaf_cap = 0;
    t->walk_cap1 = 16;
    t->short_rays = -1;
    t->walk2_min = -1;
    t->fuse_short = 1;
    t->time_march = 0;
    t->short_leaves = xb::kShortLeaves;
    t->short_samples = (int32_t)xb::kShortSamples;
    t->grab_div = 4;
    t->grab_fixed = 0;
}

int xb_tuning_get(xb_tuning* t) {
    return guarded([&] {
        XB_CHECK(t, XB_ERR_ARG, "null tuning");
        *t = tuning_snapshot();
    });
}

int xb_tuning_set(const xb_tuning* t) {
    return guarded([&] {
        xb_tuning n;
        if (t) n = *t; else xb_tuning_defaults(&n);
        XB_CHECK(n.kernel == 0 || n.kernel == 1, XB_ERR_ARG, "tuning.kernel must be 0 or 1");
        XB_CHECK(n.traversal == 0 || n.traversal == 1, XB_ERR_ARG, "tuning.traversal must be 0 or 1");
        XB_CHECK(n.leaf_cap >= 0 && n.leaf_cap <= 4096, XB_ERR_ARG, "tuning.leaf_cap out of range");
        XB_CHECK(n.walk_cap1 >= 1, XB_ERR_ARG, "tuning.walk_cap1 must be >= 1");
        XB_CHECK(n.short_rays >= -1 && n.short_rays <= 1, XB_ERR_ARG, "tuning.short_rays must be -1, 0 or 1");
        XB_CHECK(n.short_leaves >= 1 && n.short_samples >= 1, XB_ERR_ARG, "tuning.short_leaves / short_samples must be >= 1");
        XB_CHECK(n.grab_div >= 1 && n.grab_fixed >= 0 && n.grab_fixed <= 32, XB_ERR_ARG,
                 "tuning.grab_div must be >= 1 and grab_fixed in [0, 32]");
        std::lock_guard<std::mutex> g(g_tuning_mu);
        g_tuning = n;
    });
}

int xb_render(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* vol, const xb_active* iso,
              const xb_camera* cam, const xb_march* mp, int32_t tile_rank, int32_t tile_world, void* rgba8,
              double* rgba_f64, int32_t* px_counts, int64_t* stats, int32_t count_bytes, void* stream) {
    return guarded([&] {
        XB_CHECK(m && r && vol, XB_ERR_ARG, "null model, regions or volume active set");
        XB_CHECK(cam && mp && rgba8, XB_ERR_ARG, "null camera, params or output");
        XB_CHECK(cam->width >= 1 && cam->height >= 1, XB_ERR_ARG, "image must be at least 1x1 pixel");
        XB_CHECK(tile_world >= 1 && tile_rank >= 0 && tile_rank < tile_world, XB_ERR_ARG, "bad tile rank/world");
        const xb_tuning T = tuning_snapshot();
        xb::DeviceGuard g(m->m.device);
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t frame_px = (int64_t)cam->width * cam->height;
        if (tile_world == 1 && !rgba_f64 && !px_counts && frame_px > kBandSlots) {
            // Large frames render as interleaved tile bands of <= kBandSlots pixels (the
            // multi-GPU tile split, on one device), so the per-pixel walk scratch (~1 KB per
            // pixel in flight) stays bounded whatever the resolution; then one unpack.
            const int bands = (int)((frame_px + kBandSlots - 1) / kBandSlots);
            const int64_t tpr = tiles_for_rank(cam->width, cam->height, 0, bands, nullptr, nullptr);
            const int64_t band_px = tpr * xb::kTileW * xb::kTileH;
            OutBuf<uchar4> img;
            img.setup((uchar4*)rgba8, (size_t)frame_px, s);
            uchar4* packed = nullptr;
            int64_t* dst = nullptr;
            XB_CUDA(cudaMallocAsync((void**)&packed, (size_t)bands * band_px * sizeof(uchar4), s));
            XB_CUDA(cudaMallocAsync((void**)&dst, (size_t)bands * 3 * sizeof(int64_t), s));
            for (int b = 0; b < bands; b++) {
                const int rc = xb_render(m, r, field, vol, iso, cam, mp, b, bands, packed + (size_t)b * band_px,
                                         nullptr, nullptr, dst + 3 * b, count_bytes, stream);
                if (rc != XB_OK) throw xb::Error(rc, g_err);
            }
            int tx, ty;
            tiles_for_rank(cam->width, cam->height, 0, 1, &tx, &ty);
            xb::launch_unpack(packed, tpr, bands, tx, ty, cam->width, cam->height, img.dev, s);
            img.finish();
            std::vector<int64_t> hs((size_t)bands * 3);
            if (stats) XB_CUDA(cudaMemcpyAsync(hs.data(), dst, hs.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            XB_CUDA(cudaFreeAsync(packed, s));
            XB_CUDA(cudaFreeAsync(dst, s));
            XB_CUDA(cudaStreamSynchronize(s));
            if (stats) {
                stats[0] = stats[1] = stats[2] = 0;
                for (int b = 0; b < bands; b++)
                    for (int q = 0; q < 3; q++) stats[q] += hs[3 * b + q];
            }
            return;
        }
        xb::RenderArgs* A = new xb::RenderArgs();  // 8.6 KB: keep off the stack
        std::unique_ptr<xb::RenderArgs> hold(A);
        A->S = scene_view(m, r, field);
        check_active(vol, r, "volume");
        A->vflags = vol->a.flags.p;
        A->vmask4 = vol->a.mask4.p;
        XB_CHECK(!mp->use_tree || m->m.n_tree > 0, XB_ERR_NO_TREE,
                 "cell-location sampling requires a model with the split tree");
        A->use_lbvh = T.traversal == 1;
        if (A->use_lbvh) {
            A->vlb = xb::active_lbvh(r->r, vol->a, s).view();
            A->ilb = (mp->iso_on && iso) ? xb::active_lbvh(r->r, iso->a, s).view() : A->vlb;
        }
        // one thread per pixel for the LBVH traversal and the cell-location gather
        A->kernel = (T.kernel == 1 || A->use_lbvh || mp->use_tree) ? 1 : 0;
        A->vqmin = vol->a.qmin.n ? vol->a.qmin.p : nullptr;
        A->wflags = A->vflags;
        A->wmask4 = A->vmask4;
        A->wqmin = A->vqmin;
        A->walk_iso = 0;
        fill_march(A->M, mp);
        A->M.iso_on = (mp->iso_on && iso) ? 1 : 0;
        if (A->M.iso_on) check_active(iso, r, "iso");
        A->iflags = A->M.iso_on ? iso->a.flags.p : vol->a.flags.p;
        A->imask4 = A->M.iso_on ? iso->a.mask4.p : vol->a.mask4.p;
        A->W = cam->width;
        A->H = cam->height;
        for (int a = 0; a < 3; a++) {
            A->pos[a] = cam->position[a];
            A->right[a] = cam->right[a];
            A->up[a] = cam->up[a];
            A->fwd[a] = cam->forward[a];
        }
        A->tan_half = cam->tan_half;
        A->aspect = cam->aspect;
        std::memcpy(A->tf, mp->tf_rgba, sizeof(A->tf));
        int tx, ty;
        const int64_t n_local = tiles_for_rank(cam->width, cam->height, tile_rank, tile_world, &tx, &ty);
        A->tiles_x = tx;
        A->tiles_y = ty;
        A->tile_rank = tile_rank;
        A->tile_world = tile_world;
        A->packed = tile_world > 1;
        const size_t npx = A->packed ? (size_t)n_local * xb::kTileW * xb::kTileH : (size_t)cam->width * cam->height;
        OutBuf<uchar4> o8;
        OutBuf<double4> of;
        OutBuf<int2> oc;
        o8.setup((uchar4*)rgba8, npx, s);
        of.setup((double4*)rgba_f64, rgba_f64 ? npx : 0, s);
        oc.setup((int2*)px_counts, px_counts ? npx : 0, s);
        A->out8 = o8.dev;
        A->outf = of.dev;
        A->outcnt = oc.dev;
        // per-call scratch (stream-ordered pool): [regions, samples, bytes, work counter, list lengths x5,
        // debug counters x7, short-ray grab counter]
        unsigned long long* scratch = nullptr;
        XB_CUDA(cudaMallocAsync((void**)&scratch, 32 * sizeof(unsigned long long), s));
        XB_CUDA(cudaMemsetAsync(scratch, 0, 32 * sizeof(unsigned long long), s));
        A->walk_counter = scratch + 4;
        unsigned long long* dstats = (stats || count_bytes) ? scratch : nullptr;
        A->stats = dstats;
        A->work_counter = scratch + 3;
        A->dbg = xb::kDebugChunks ? scratch + 9 : nullptr;  // [9, 16): make DEBUG_CHUNKS=1 builds only
        A->short_counter = scratch + 16;
        A->fuse_short = T.fuse_short != 0;
        A->grab_div = T.grab_div;
        A->grab_fixed = T.grab_fixed;
        double* iso_buf = nullptr;
        if (A->M.iso_on) {
            const size_t n_slots = (size_t)n_local * xb::kTileW * xb::kTileH;
            XB_CUDA(cudaMallocAsync((void**)&iso_buf, 2 * std::max<size_t>(n_slots, 1) * sizeof(double), s));
            A->iso_tend = iso_buf;
            A->iso_shade = iso_buf + n_slots;
        }
        // k_walk -> k_warp leaf lists (the default pipeline; tuning.walk_lists = 0 runs k_warp's
        // frontier-only path)
        int32_t* leaf_buf = nullptr;
        A->leaves = nullptr;
        A->leaf_count = nullptr;
        A->short_list = nullptr;
        A->long_list = nullptr;
        A->any_list = nullptr;
        A->short_min = 0;
        A->walk_cap1 = 0;
        A->walk2_min = 0;
        A->cut_list = nullptr;
        A->short_leaves = T.short_leaves;
        A->short_samples = (float)T.short_samples;
        A->leaf_cap = 0;
        A->cut_tau = 1;
        if (A->kernel == 0 && T.walk_lists) {
            keep_pool(m->m.device);
            // Leaf cap per walk (then k_warp resumes the rest).  Single-pass sweep with resume,
            // ms/frame (round-1 pipeline):
            //   cap      16    32    48    64    96    128
            //   C2     7.54  7.08  6.81  6.62  6.42  6.47     (357K candidate rays, ~46 visits each)
            //   C3     1.48  1.52  1.57  1.61  1.76  1.98     (312K candidates, ~6 visits, long tail)
            //   C5                 3.37        3.40           (272K candidates)
            // C3's few very long walks set k_walk's length; C2's many long walks are cheaper in
            // k_walk than in the frontier.  Neither the candidate count (similar in all three) nor a
            // clock budget per walk (C2 +15-25 %) separates them: hence the two passes below
            // (16 leaves, then k_walk2 to 96 when many walks were cut).
            const int cap = T.leaf_cap > 0 ? T.leaf_cap : 96;
            const size_t n_slots = (size_t)n_local * xb::kTileW * xb::kTileH;
            const size_t ns1 = std::max<size_t>(n_slots, 1);
            const size_t res_words = 1 + 3 * xb::kResume;
            const size_t nblk = (ns1 + xb::kWalkThreads - 1) / xb::kWalkThreads;
            XB_CUDA(cudaMallocAsync((void**)&leaf_buf, (ns1 * (cap + 6 + res_words) + 3 * nblk) * sizeof(int32_t), s));
            A->leaf_count = leaf_buf;
            A->hit_list = leaf_buf + ns1;
            // two-pass walk: pass 1 caps at 16 leaves; pass 2 continues the cap-cut walks to the
            // list capacity (96) when there are >= 500 x SMs of them.  tools/ab.py, ms (C3 / C2 /
            // C5): single cap 64: 1.39 / 6.72 / 3.45; 24+96: 1.22 / 6.54 / 3.75; 16+96: 1.20 /
            // 6.55 / 3.64; 16+64: 1.19 / 6.73 / 3.51.
            A->walk_cap1 = T.leaf_cap > 0 ? cap : std::min(cap, std::max(1, T.walk_cap1));
            A->cut_list = leaf_buf + (3 + res_words + cap) * ns1;
            A->long_list = leaf_buf + (4 + res_words + cap) * ns1;
            A->any_list = leaf_buf + (5 + res_words + cap) * ns1;
            A->blk_counts = leaf_buf + (6 + res_words + cap) * ns1;
            // short rays (<= 8 leaves, <= 24 estimated samples) run one per lane, used only when the
            // frame has >= 1000 x SMs of them (decided on the device).  tools/ab.py, ms, forced on
            // vs off: C3 (270K short rays) 1.56 vs 1.61, C5 (44K) 3.70 vs 3.40, C2 (57K) 6.82 vs
            // 6.66 — one thread per ray pays only when short rays are plentiful.
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->m.device);
            A->short_list = T.short_rays == 0 ? nullptr : leaf_buf + 2 * ns1;
            A->short_min = T.short_rays == 1 ? 0 : 1000ll * sms;
            A->walk2_min = T.walk2_min >= 0 ? T.walk2_min : 500ll * sms;
            A->resume = leaf_buf + 3 * ns1;
            A->leaves = leaf_buf + (3 + res_words) * ns1;
            A->leaf_cap = cap;
        }
        MarchEvents me{m->m.device, {nullptr, nullptr}};
        A->march_events = nullptr;
        if (T.time_march && A->kernel == 0) {
            XB_CUDA(cudaEventCreate(&me.ev[0]));
            XB_CUDA(cudaEventCreate(&me.ev[1]));
            A->march_events = me.ev;
        }
        int32_t* fixup_buf = nullptr;  // k_warp's pixels for the exact FP64 shading re-render (k_fixup)
        if (A->kernel == 0 && A->M.grad_mode == 1) {
            const size_t n_slots = std::max<size_t>((size_t)n_local * xb::kTileW * xb::kTileH, 1);
            XB_CUDA(cudaMallocAsync((void**)&fixup_buf, n_slots * sizeof(int32_t), s));
            A->fixup_list = fixup_buf;
            A->fixup_count = scratch + 19;  // zeroed with the scratch
        }
        xb::launch_render(*A, n_local, count_bytes != 0, s);
        if (fixup_buf) XB_CUDA(cudaFreeAsync(fixup_buf, s));
        if (A->march_events) {
            std::lock_guard<std::mutex> eg(g_events_mu);
            g_events.push_back(me);
        }
        if (A->dbg) {
            unsigned long long d[20];
            XB_CUDA(cudaMemcpyAsync(d, A->dbg, sizeof d, cudaMemcpyDeviceToHost, s));
            XB_CUDA(cudaStreamSynchronize(s));
            fprintf(stderr, "xb_render: k_warp %llu rays, %llu samples, %llu regions, %llu chunks, %.1f lanes/chunk, "
                            "%.2f bricks/sample, %.2f max bricks/chunk\n",
                    d[2], d[3], d[4], d[0], d[0] ? (double)d[1] / (double)d[0] : 0.0,
                    d[1] ? (double)d[5] / (double)d[1] : 0.0, d[0] ? (double)d[6] / (double)d[0] : 0.0);
            fprintf(stderr, "xb_render: k_warp warp-cycles: long phase %.3g (rays %.3g, chunks %.3g), short phase %.3g\n",
                    (double)d[19], (double)d[17], (double)d[16], (double)d[18]);
        }
        if (leaf_buf) XB_CUDA(cudaFreeAsync(leaf_buf, s));
        if (iso_buf) XB_CUDA(cudaFreeAsync(iso_buf, s));
        o8.finish();
        of.finish();
        oc.finish();
        unsigned long long hs[3] = {0, 0, 0};
        const bool dev_stats = stats && is_device_ptr(stats);  // device counters: no host synchronisation
        if (dev_stats) XB_CUDA(cudaMemcpyAsync(stats, dstats, sizeof hs, cudaMemcpyDeviceToDevice, s));
        else if (dstats) XB_CUDA(cudaMemcpyAsync(hs, dstats, sizeof hs, cudaMemcpyDeviceToHost, s));
        XB_CUDA(cudaFreeAsync(scratch, s));
        const bool host_out = o8.owned || of.owned || oc.owned || (dstats && !dev_stats);
        if (host_out) XB_CUDA(cudaStreamSynchronize(s));
        if (stats && !dev_stats) {
            stats[0] = (int64_t)hs[0];
            stats[1] = (int64_t)hs[1];
            stats[2] = (int64_t)hs[2];
        }
    });
}

int xb_unpack_tiles(const void* packed, int64_t tiles_per_rank, int32_t world, int32_t width, int32_t height,
                    void* rgba8, void* stream) {
    return guarded([&] {
        XB_CHECK(packed && rgba8 && world >= 1, XB_ERR_ARG, "bad unpack arguments");
        const int tx = (width + xb::kTileW - 1) / xb::kTileW, ty = (height + xb::kTileH - 1) / xb::kTileH;
        xb::launch_unpack((const uchar4*)packed, tiles_per_rank, world, tx, ty, width, height, (uchar4*)rgba8,
                          (cudaStream_t)stream);
    });
}

static int run_rays(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* act, const xb_march* mp,
                    int mode, int64_t n, const double* o, const double* d, const double* t0, const double* t1,
                    const double* rho, double* out, int64_t* counts) {
    return guarded([&] {
        XB_CHECK(mp && n >= 0, XB_ERR_ARG, "bad ray batch");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        auto B = std::make_unique<xb::RayBatchArgs>();
        B->S = scene_view(m, r, field);
        check_active(act, r, mode == 0 ? "volume" : "iso");
        B->vflags = act->a.flags.p;
        B->iflags = act->a.flags.p;
        fill_march(B->M, mp);
        B->mode = mode;
        B->use_lbvh = tuning_snapshot().traversal == 1;
        if (B->use_lbvh) B->vlb = B->ilb = xb::active_lbvh(r->r, act->a, st.s).view();
        B->n = n;
        std::memcpy(B->tf, mp->tf_rgba, sizeof(B->tf));
        xb::DevBuf<double> dO, dD, d0, d1, dr, dout;
        xb::DevBuf<int64_t> dc;
        dO.upload(o, 3 * n, st.s);
        dD.upload(d, 3 * n, st.s);
        d0.upload(t0, n, st.s);
        d1.upload(t1, n, st.s);
        dr.upload(rho, n, st.s);
        dout.alloc(4 * n + 1);
        dc.alloc(2 * n + 1);
        B->o = dO.p; B->d = dD.p; B->t0 = d0.p; B->t1 = d1.p; B->rho = dr.p; B->out = dout.p; B->counts = dc.p;
        xb::launch_rays(*B, st.s);
        dout.download(out, 4 * n, st.s);
        dc.download(counts, 2 * n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_integrate_rays(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* vol,
                      const xb_march* mp, int64_t n, const double* o, const double* d, const double* t0,
                      const double* t1, const double* rho, double* out, int64_t* counts) {
    return run_rays(m, r, field, vol, mp, 0, n, o, d, t0, t1, rho, out, counts);
}

int xb_iso_rays(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* iso, const xb_march* mp,
                int64_t n, const double* o, const double* d, const double* t0, const double* t1, const double* rho,
                double* out, int32_t* hit) {
    std::vector<int64_t> c(2 * std::max<int64_t>(n, 1));
    int rc = run_rays(m, r, field, iso, mp, 1, n, o, d, t0, t1, rho, out, c.data());
    if (rc == XB_OK)
        for (int64_t q = 0; q < n; q++) hit[q] = (int32_t)c[2 * q];
    return rc;
}

int xb_sample_points(const xb_model* m, const xb_regions* r, int32_t field, int64_t n, const double* p,
                     const int32_t* region, int32_t want_grad, int32_t* region_out, double* acc) {
    return guarded([&] {
        XB_CHECK(n >= 0, XB_ERR_ARG, "bad point count");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        const xb::SceneView S = scene_view(m, r, field);
        xb::DevBuf<double> dp, dacc;
        xb::DevBuf<int32_t> drin, drout;
        dp.upload(p, 3 * n, st.s);
        if (region) drin.upload(region, n, st.s);
        drout.alloc(n + 1);
        dacc.alloc(9 * n + 1);
        xb::sample_points(S, n, dp.p, region ? drin.p : nullptr, want_grad, drout.p, dacc.p, st.s);
        drout.download(region_out, n, st.s);
        dacc.download(acc, 9 * n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_sample_scan(const xb_model* m, int32_t field, int64_t n, const double* p, double* out) {
    return guarded([&] {
        XB_CHECK(m && n >= 0, XB_ERR_ARG, "bad arguments");
        XB_CHECK(field >= 0 && field < m->m.n_fields, XB_ERR_ARG, "field index out of range");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        xb::SceneView S{};
        S.brick_a = m->m.brick_a.p;
        S.brick_m = m->m.brick_m.p;
        S.vals = m->m.vals.p + (size_t)field * (size_t)m->m.n_cells;
        xb::DevBuf<double> dp, dout;
        dp.upload(p, 3 * n, st.s);
        dout.alloc(2 * n + 1);
        xb::sample_scan(S, m->m.n_bricks, n, dp.p, dout.p, st.s);
        dout.download(out, 2 * n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_sample_scan_cells(const xb_cells* c, int64_t n, const double* p, double* out) {
    return guarded([&] {
        XB_CHECK(c && n >= 0, XB_ERR_ARG, "bad arguments");
        xb::DeviceGuard g(c->c.device);
        OwnedStream st;
        xb::DevBuf<double> dp, dout;
        dp.upload(p, 3 * n, st.s);
        dout.alloc(2 * n + 1);
        xb::scan_cells(c->c.i.p, c->c.j.p, c->c.k.p, c->c.level.p, c->c.vals.p, c->c.n, n, dp.p, dout.p, st.s);
        dout.download(out, 2 * n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_trace_intervals(const xb_model* m, const xb_regions* r, const xb_active* a, int64_t n, const double* o,
                       const double* d, double t_start, double t_max, int32_t cap, double* t_in, double* t_out,
                       int32_t* region, int32_t* count) {
    return guarded([&] {
        XB_CHECK(n >= 0 && cap >= 0, XB_ERR_ARG, "bad trace arguments");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        const xb::SceneView S = scene_view(m, r, 0);
        check_active(a, r, "trace");
        xb::DevBuf<double> dO, dD, di, dq;
        xb::DevBuf<int32_t> dr, dc;
        dO.upload(o, 3 * n, st.s);
        dD.upload(d, 3 * n, st.s);
        di.alloc((size_t)n * cap + 1);
        dq.alloc((size_t)n * cap + 1);
        dr.alloc((size_t)n * cap + 1);
        dc.alloc(n + 1);
        xb::trace_intervals(S, a->a.flags.p, n, dO.p, dD.p, t_start, t_max, cap, di.p, dq.p, dr.p, dc.p, st.s);
        di.download(t_in, (size_t)n * cap, st.s);
        dq.download(t_out, (size_t)n * cap, st.s);
        dr.download(region, (size_t)n * cap, st.s);
        dc.download(count, n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

// ---- LBVH (RegionBvh node arrays, closest-hit / point queries) ----

int xb_active_lbvh_info(const xb_active* a, int64_t* n_nodes, int32_t* depth, double* build_ms) {
    return guarded([&] {
        XB_CHECK(a != nullptr && a->owner != nullptr, XB_ERR_ARG, "null active set");
        xb::DeviceGuard g(a->a.device);
        OwnedStream st;
        const xb::DevLbvh& L = xb::active_lbvh(a->owner->r, a->a, st.s);
        if (n_nodes) *n_nodes = L.n_prims ? 2 * L.n_prims - 1 : 1;
        if (depth) *depth = L.depth;
        if (build_ms) *build_ms = L.build_ms;
    });
}

int xb_active_lbvh_download(const xb_active* a, double* node_lo, double* node_hi, int32_t* left, int32_t* right,
                            int64_t* start, int32_t* count, int32_t* prims) {
    return guarded([&] {
        XB_CHECK(a != nullptr && a->owner != nullptr, XB_ERR_ARG, "null active set");
        xb::DeviceGuard g(a->a.device);
        OwnedStream st;
        const xb::DevLbvh& L = xb::active_lbvh(a->owner->r, a->a, st.s);
        const int64_t n = L.n_prims;
        if (n == 0) {  // the reference's dummy node (R/accel.py:205-212)
            for (int c = 0; c < 3; c++) {
                node_lo[c] = INFINITY;
                node_hi[c] = -INFINITY;
            }
            left[0] = right[0] = -1;
            start[0] = 0;
            count[0] = 0;
            return;
        }
        std::vector<xb::LbvhNode> nodes(std::max<int64_t>(n - 1, 0));
        std::vector<xb::RegionRec> rec(a->owner->r.n_regions);
        std::vector<int32_t> pr(n);
        if (n > 1) L.nodes.download(nodes.data(), n - 1, st.s);
        L.prims.download(pr.data(), n, st.s);
        a->owner->r.rec.download(rec.data(), rec.size(), st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
        // internal node i -> i, leaf k -> (n - 1) + k; leaves hold one region (start k, count 1)
        auto node_of = [&](int32_t c) -> int64_t { return c >= 0 ? c : (n - 1) + (int64_t)(~c); };
        for (int64_t i = 0; i < n - 1; i++) {
            for (int c = 0; c < 3; c++) {
                node_lo[3 * i + c] = nodes[i].lo[c] * 0.5;
                node_hi[3 * i + c] = nodes[i].hi[c] * 0.5;
            }
            left[i] = (int32_t)node_of(nodes[i].left);
            right[i] = (int32_t)node_of(nodes[i].right);
            start[i] = 0;
            count[i] = 0;
        }
        for (int64_t k = 0; k < n; k++) {
            const int64_t i = n - 1 + k;
            const xb::RegionRec& rr = rec[pr[k]];
            for (int c = 0; c < 3; c++) {
                node_lo[3 * i + c] = rr.lo[c] * 0.5;
                node_hi[3 * i + c] = rr.hi[c] * 0.5;
            }
            left[i] = right[i] = -1;
            start[i] = k;
            count[i] = 1;
            prims[k] = pr[k];
        }
    });
}

int xb_trace_intervals_lbvh(const xb_model* m, const xb_regions* r, const xb_active* a, int64_t n, const double* o,
                            const double* d, double t_start, double t_max, int32_t cap, double* t_in, double* t_out,
                            int32_t* region, int32_t* count) {
    return guarded([&] {
        XB_CHECK(n >= 0 && cap >= 0, XB_ERR_ARG, "bad trace arguments");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        const xb::SceneView S = scene_view(m, r, 0);
        check_active(a, r, "trace");
        const xb::LbvhView L = xb::active_lbvh(r->r, a->a, st.s).view();
        xb::DevBuf<double> dO, dD, di, dq;
        xb::DevBuf<int32_t> dr, dc;
        dO.upload(o, 3 * n, st.s);
        dD.upload(d, 3 * n, st.s);
        di.alloc((size_t)n * cap + 1);
        dq.alloc((size_t)n * cap + 1);
        dr.alloc((size_t)n * cap + 1);
        dc.alloc(n + 1);
        xb::trace_intervals(S, a->a.flags.p, n, dO.p, dD.p, t_start, t_max, cap, di.p, dq.p, dr.p, dc.p, st.s, &L);
        di.download(t_in, (size_t)n * cap, st.s);
        dq.download(t_out, (size_t)n * cap, st.s);
        dr.download(region, (size_t)n * cap, st.s);
        dc.download(count, n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

int xb_point_query_lbvh(const xb_model* m, const xb_regions* r, const xb_active* a, int64_t n, const double* p,
                        int32_t* region) {
    return guarded([&] {
        XB_CHECK(n >= 0, XB_ERR_ARG, "bad point count");
        xb::DeviceGuard g(m->m.device);
        OwnedStream st;
        const xb::SceneView S = scene_view(m, r, 0);
        check_active(a, r, "point query");
        const xb::LbvhView L = xb::active_lbvh(r->r, a->a, st.s).view();
        xb::DevBuf<double> dp;
        xb::DevBuf<int32_t> dr(n + 1);
        dp.upload(p, 3 * n, st.s);
        xb::point_query_lbvh(S, L, n, dp.p, dr.p, st.s);
        dr.download(region, n, st.s);
        XB_CUDA(cudaStreamSynchronize(st.s));
    });
}

}  // extern "C"
