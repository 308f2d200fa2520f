// accel.cuh — active sets and point / interval queries.
#pragma once
#include <memory>
#include <mutex>
#include "lbvh.cuh"

namespace xb {

// An active region set + its k-d subtree flags: the B200 form of the
// reference's pruned RegionBvh (R/accel.py:125-155).
struct DevActive {
    int device = 0;
    int kind = 0;  // 0 volume (max_opacity > 0), 1 iso (lo <= iso <= hi), 2 all regions
    int64_t n_active = 0;
    DevBuf<uint8_t> act;     // per region
    DevBuf<uint8_t> flags;   // per k-d node
    DevBuf<uint8_t> mask4;   // per Kd4 node: active bit per child slot
    DevBuf<float> qmin;      // volume sets: per-region opacity minorant (optical depth per unit length at spc 1)
    DevBuf<int32_t> prims;   // ascending active region ids
    double build_ms = 0.0;
    // LBVH over the active regions (RegionBvh node arrays / closest-hit queries), built on first use
    mutable std::mutex lb_mu;
    mutable std::unique_ptr<DevLbvh> lb;
};

const DevLbvh& active_lbvh(const DevRegions& R, const DevActive& a, cudaStream_t s);

void build_kd4(DevRegions& R, cudaStream_t s);
void build_kd4_mask(const DevRegions& R, const uint8_t* flags, DevBuf<uint8_t>& mask, cudaStream_t s);

void build_active(const DevRegions& R, int kind, int field, double tf_lo, double tf_hi, const double* rgba_host,
                  double iso, DevActive& out, cudaStream_t s);

void sample_points(const SceneView& S, int64_t n, const double* p, const int32_t* rid_in, int want_grad, int32_t* rid_out,
                   double* out, cudaStream_t s);
void scan_cells(const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* l, const float* v, int64_t n_cells,
                int64_t n, const double* p, double* out, cudaStream_t s);
void sample_scan(const SceneView& S, int64_t n_bricks, int64_t n, const double* p, double* out, cudaStream_t s);
void trace_intervals(const SceneView& S, const uint8_t* flags, int64_t n, const double* o, const double* d, double t0,
                     double t1, int cap, double* tin, double* tout, int32_t* reg, int32_t* cnt, cudaStream_t s,
                     const LbvhView* lb = nullptr);
void point_query_lbvh(const SceneView& S, const LbvhView& L, int64_t n, const double* p, int32_t* out, cudaStream_t s);

}  // namespace xb
