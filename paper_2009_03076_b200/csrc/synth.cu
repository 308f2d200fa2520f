// synth.cu — GPU restatement of the reference's synthetic AMR generator
// (`generate_synthetic`, R/io.py:247-295, fields R/io.py:120-195) for the
// 10^8-10^9-cell configurations, where
// the numpy path takes minutes.  Same top-down octree refinement, same cell
// order (levels max..0; within a level, parents in order, children x fastest
// then y then z), same FP64 expressions; transcendental functions are CUDA's
// (exp/sin/cos within 1-2 ulp of numpy's), so a refinement decision or an
// f32 value can differ only where the FP64 result sits within an ulp of the
// threshold or of an f32 rounding boundary (tests/test_gpu_parity.py pins
// the generator cell-for-cell against the reference's own output).
#include "../../include/exabricks.h"
#include "common.cuh"
#include "scan.cuh"
#include "synth.cuh"

namespace xb {
namespace {

constexpr int BS = 256;

struct Field {
    int kind;
    double c[3], sigma, amp;   // gaussian
    double dir[3], offset;     // ramp
    double constant;           // constant
    int n_waves;
    double waves[8][5];        // octaves: k[3], phase, amp
};

struct Spheres {
    int n;
    double s[32][4];
};

__device__ __forceinline__ double f_value(const Field& F, double x, double y, double z) {
    if (F.kind == 0) {  // GaussianField.value: amp * exp(-d2 / (2 * sigma**2))
        const double dx = x - F.c[0], dy = y - F.c[1], dz = z - F.c[2];
        const double d2 = (dx * dx + dy * dy) + dz * dz;
        return F.amp * exp(-d2 / (2.0 * (F.sigma * F.sigma)));
    }
    if (F.kind == 1) return ((x * F.dir[0] + y * F.dir[1]) + z * F.dir[2]) + F.offset;  // RampField
    if (F.kind == 2) return F.constant;                                                  // ConstantField
    double out = 0.0;                                                                    // OctaveField
    for (int w = 0; w < F.n_waves; w++) {
        const double* k = F.waves[w];
        out += k[4] * sin(((x * k[0] + y * k[1]) + z * k[2]) + k[3]);
    }
    return out;
}

// |grad f| (np.linalg.norm(gradient, axis=1))
__device__ __forceinline__ double f_gradnorm(const Field& F, double x, double y, double z) {
    double g0, g1, g2;
    if (F.kind == 0) {  // -d * (v / sigma**2)
        const double v = f_value(F, x, y, z);
        const double s = v / (F.sigma * F.sigma);
        g0 = -(x - F.c[0]) * s;
        g1 = -(y - F.c[1]) * s;
        g2 = -(z - F.c[2]) * s;
    } else if (F.kind == 1) {
        g0 = F.dir[0]; g1 = F.dir[1]; g2 = F.dir[2];
    } else if (F.kind == 2) {
        g0 = g1 = g2 = 0.0;
    } else {
        g0 = g1 = g2 = 0.0;
        for (int w = 0; w < F.n_waves; w++) {
            const double* k = F.waves[w];
            const double a = k[4] * cos(((x * k[0] + y * k[1]) + z * k[2]) + k[3]);
            g0 += a * k[0];
            g1 += a * k[1];
            g2 += a * k[2];
        }
    }
    return sqrt((g0 * g0 + g1 * g1) + g2 * g2);
}

// _in_spheres: sum((c - centre)**2) < r * r for any sphere
__device__ __forceinline__ bool in_spheres(const Spheres& S, double x, double y, double z) {
    for (int q = 0; q < S.n; q++) {
        const double dx = x - S.s[q][0], dy = y - S.s[q][1], dz = z - S.s[q][2];
        if ((dx * dx + dy * dy) + dz * dz < S.s[q][3] * S.s[q][3]) return true;
    }
    return false;
}

__global__ void k_fill(int64_t n, int32_t* a, int32_t v) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c < n) a[c] = v;
}

__global__ void k_init(int64_t n, int64_t g1, int64_t g2, int top, int32_t* i, int32_t* j, int32_t* k) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;  // meshgrid(indexing="ij").ravel(): gi slowest, gk fastest
    i[c] = (int32_t)((c / (g1 * g2)) * top);
    j[c] = (int32_t)(((c / g2) % g1) * top);
    k[c] = (int32_t)((c % g2) * top);
}

__global__ void k_fire(int64_t n, const int32_t* __restrict__ i, const int32_t* __restrict__ j,
                       const int32_t* __restrict__ k, int w, double thr, const Field F, const Spheres R,
                       int32_t* __restrict__ fire, int32_t* __restrict__ keep) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    const double h = (double)w / 2.0;
    const double x = (double)i[c] + h, y = (double)j[c] + h, z = (double)k[c] + h;
    bool f = f_gradnorm(F, x, y, z) * (double)w >= thr;
    if (R.n) f = f || in_spheres(R, x, y, z);
    fire[c] = f ? 1 : 0;
    keep[c] = f ? 0 : 1;
}

__global__ void k_split(int64_t n, const int32_t* __restrict__ i, const int32_t* __restrict__ j,
                        const int32_t* __restrict__ k, const int32_t* __restrict__ fire,
                        const int32_t* __restrict__ fpos, const int32_t* __restrict__ kpos, int w, int level,
                        int32_t* __restrict__ ni, int32_t* __restrict__ nj, int32_t* __restrict__ nk,
                        int32_t* __restrict__ oi, int32_t* __restrict__ oj, int32_t* __restrict__ ok,
                        int32_t* __restrict__ ol) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    if (fire[c]) {
        const int h = w / 2;
        const int64_t b = 8 * (int64_t)fpos[c];
        for (int q = 0; q < 8; q++) {  // _CHILD order: x fastest, then y, then z
            ni[b + q] = i[c] + (q & 1) * h;
            nj[b + q] = j[c] + ((q >> 1) & 1) * h;
            nk[b + q] = k[c] + ((q >> 2) & 1) * h;
        }
    } else {
        const int64_t p = kpos[c];
        oi[p] = i[c];
        oj[p] = j[c];
        ok[p] = k[c];
        ol[p] = level;
    }
}

__global__ void k_hole_keep(int64_t n, const int32_t* __restrict__ i, const int32_t* __restrict__ j,
                            const int32_t* __restrict__ k, const int32_t* __restrict__ l, const Spheres H,
                            int32_t* __restrict__ keep) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    const double h = (double)(1 << l[c]) / 2.0;  // (2.0**lev) / 2
    keep[c] = in_spheres(H, (double)i[c] + h, (double)j[c] + h, (double)k[c] + h) ? 0 : 1;
}

__global__ void k_compact(int64_t n, const int32_t* __restrict__ keep, const int32_t* __restrict__ pos,
                          const int32_t* __restrict__ i, const int32_t* __restrict__ j, const int32_t* __restrict__ k,
                          const int32_t* __restrict__ l, int32_t* __restrict__ oi, int32_t* __restrict__ oj,
                          int32_t* __restrict__ ok, int32_t* __restrict__ ol) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n || !keep[c]) return;
    const int64_t p = pos[c];
    oi[p] = i[c];
    oj[p] = j[c];
    ok[p] = k[c];
    ol[p] = l[c];
}

__global__ void k_values(int64_t n, const int32_t* __restrict__ i, const int32_t* __restrict__ j,
                         const int32_t* __restrict__ k, const int32_t* __restrict__ l, const Field F,
                         float* __restrict__ v) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n) return;
    const double h = (double)(1 << l[c]) / 2.0;
    v[c] = (float)f_value(F, (double)i[c] + h, (double)j[c] + h, (double)k[c] + h);
}

Field make_field(const xb_synth_spec& sp) {
    Field F{};
    F.kind = sp.field;
    for (int a = 0; a < 3; a++) {
        F.c[a] = sp.center[a];
        F.dir[a] = sp.direction[a];
    }
    F.sigma = sp.sigma;
    F.amp = sp.amp;
    F.offset = sp.offset;
    F.constant = sp.constant;
    F.n_waves = sp.n_waves;
    for (int w = 0; w < 8; w++)
        for (int q = 0; q < 5; q++) F.waves[w][q] = sp.waves[w][q];
    return F;
}

Spheres make_spheres(int n, const double (*s)[4]) {
    Spheres S{};
    S.n = n;
    for (int q = 0; q < n; q++)
        for (int c = 0; c < 4; c++) S.s[q][c] = s[q][c];
    return S;
}

}  // namespace

void generate_synthetic_device(const xb_synth_spec& sp, int device, DevCells& out, cudaStream_t s) {
    DeviceGuard g(device);
    out = DevCells();
    out.device = device;
    XB_CHECK(sp.field >= 0 && sp.field <= 3, XB_ERR_ARG, "unknown field kind");
    XB_CHECK(sp.max_level >= 0 && sp.max_level <= 20, XB_ERR_ARG, "max_level out of range");
    XB_CHECK(sp.n_holes >= 0 && sp.n_holes <= 32 && sp.n_refine >= 0 && sp.n_refine <= 32, XB_ERR_ARG,
             "at most 32 hole / refine spheres");
    XB_CHECK(sp.n_waves >= 0 && sp.n_waves <= 8, XB_ERR_ARG, "at most 8 octaves");
    const int64_t top = 1ll << sp.max_level;
    for (int a = 0; a < 3; a++)
        XB_CHECK(sp.extent[a] > 0 && sp.extent[a] % top == 0 && sp.extent[a] < (1ll << 30), XB_ERR_ARG,
                 "extent must be positive multiples of 2**max_level");
    const Field F = make_field(sp);
    const Spheres R = make_spheres(sp.n_refine, sp.refine);
    const Spheres H = make_spheres(sp.n_holes, sp.holes);
    const int64_t g0 = sp.extent[0] / top, g1 = sp.extent[1] / top, g2 = sp.extent[2] / top;
    int64_t n = g0 * g1 * g2;
    XB_CHECK(n < (1ll << 31) - 2, XB_ERR_RANGE, "synthetic grid too large");
    DevBuf<int32_t> ci(n + 1), cj(n + 1), ck(n + 1);
    if (n) k_init<<<grid_for(n, BS), BS, 0, s>>>(n, g1, g2, (int)top, ci.p, cj.p, ck.p);
    check_launch("k_init");
    CubTemp tmp;
    // per level output segments, concatenated max_level..0 at the end
    std::vector<DevBuf<int32_t>> seg_i, seg_j, seg_k, seg_l;
    std::vector<int64_t> seg_n;
    for (int level = sp.max_level; level >= 0; level--) {
        const int w = 1 << level;
        DevBuf<int32_t> fire(n + 1), keep(n + 1), fpos(n + 1), kpos(n + 1);
        if (level > 0) {
            if (n) k_fire<<<grid_for(n, BS), BS, 0, s>>>(n, ci.p, cj.p, ck.p, w, sp.threshold, F, R, fire.p, keep.p);
            check_launch("k_fire");
        } else {  // level 0: everything left is emitted
            XB_CUDA(cudaMemsetAsync(fire.p, 0, (n + 1) * 4, s));
            if (n) k_fill<<<grid_for(n, BS), BS, 0, s>>>(n, keep.p, 1);
        }
        XB_CUDA(cudaMemsetAsync(fire.p + n, 0, 4, s));
        XB_CUDA(cudaMemsetAsync(keep.p + n, 0, 4, s));
        exclusive_sum(tmp, fire.p, fpos.p, n + 1, s);
        exclusive_sum(tmp, keep.p, kpos.p, n + 1, s);
        const int64_t n_fire = read_scalar(fpos.p + n, s), n_keep = read_scalar(kpos.p + n, s);
        XB_CHECK(8 * n_fire < (1ll << 31) - 2, XB_ERR_RANGE, "synthetic refinement exceeds 2^31 cells");
        DevBuf<int32_t> ni(8 * n_fire + 1), nj(8 * n_fire + 1), nk(8 * n_fire + 1);
        DevBuf<int32_t> oi(n_keep + 1), oj(n_keep + 1), ok(n_keep + 1), ol(n_keep + 1);
        if (n) k_split<<<grid_for(n, BS), BS, 0, s>>>(n, ci.p, cj.p, ck.p, fire.p, fpos.p, kpos.p, w, level, ni.p,
                                                  nj.p, nk.p, oi.p, oj.p, ok.p, ol.p);
        check_launch("k_split");
        seg_i.push_back(std::move(oi)); seg_j.push_back(std::move(oj));
        seg_k.push_back(std::move(ok)); seg_l.push_back(std::move(ol));
        seg_n.push_back(n_keep);
        ci = std::move(ni); cj = std::move(nj); ck = std::move(nk);
        n = 8 * n_fire;
    }
    int64_t total = 0;
    for (int64_t m : seg_n) total += m;
    XB_CHECK(total < (1ll << 31) - 2, XB_ERR_RANGE, "synthetic model exceeds 2^31 cells");
    DevBuf<int32_t> ai(total + 1), aj(total + 1), ak(total + 1), al(total + 1);
    int64_t off = 0;
    for (size_t q = 0; q < seg_n.size(); q++) {
        const size_t b = seg_n[q] * sizeof(int32_t);
        if (b) {
            XB_CUDA(cudaMemcpyAsync(ai.p + off, seg_i[q].p, b, cudaMemcpyDeviceToDevice, s));
            XB_CUDA(cudaMemcpyAsync(aj.p + off, seg_j[q].p, b, cudaMemcpyDeviceToDevice, s));
            XB_CUDA(cudaMemcpyAsync(ak.p + off, seg_k[q].p, b, cudaMemcpyDeviceToDevice, s));
            XB_CUDA(cudaMemcpyAsync(al.p + off, seg_l[q].p, b, cudaMemcpyDeviceToDevice, s));
        }
        off += seg_n[q];
    }
    seg_i.clear(); seg_j.clear(); seg_k.clear(); seg_l.clear();
    if (H.n && total) {  // holes drop emitted cells whose centre lies inside (stable)
        DevBuf<int32_t> keep(total + 1), pos(total + 1);
        k_hole_keep<<<grid_for(total, BS), BS, 0, s>>>(total, ai.p, aj.p, ak.p, al.p, H, keep.p);
        XB_CUDA(cudaMemsetAsync(keep.p + total, 0, 4, s));
        exclusive_sum(tmp, keep.p, pos.p, total + 1, s);
        const int64_t kept = read_scalar(pos.p + total, s);
        DevBuf<int32_t> bi(kept + 1), bj(kept + 1), bk(kept + 1), bl(kept + 1);
        k_compact<<<grid_for(total, BS), BS, 0, s>>>(total, keep.p, pos.p, ai.p, aj.p, ak.p, al.p, bi.p, bj.p, bk.p,
                                                     bl.p);
        check_launch("k_compact");
        ai = std::move(bi); aj = std::move(bj); ak = std::move(bk); al = std::move(bl);
        total = kept;
    }
    out.n = total;
    out.vals.alloc(total + 1);
    if (total) k_values<<<grid_for(total, BS), BS, 0, s>>>(total, ai.p, aj.p, ak.p, al.p, F, out.vals.p);
    check_launch("k_values");
    out.i = std::move(ai); out.j = std::move(aj); out.k = std::move(ak); out.level = std::move(al);
    XB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace xb
