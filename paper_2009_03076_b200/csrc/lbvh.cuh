// lbvh.cuh — linear BVH over active region boxes (Morton order + Karras 2012
// hierarchy, csrc/lbvh.cu); the node layout and the software traversal
// (`lbvh_next_hit`, `lbvh_point`) live in march.cuh.  The B200 form of the
// reference's RegionBvh / _bvh_next_hit / _bvh_point_query (R/accel.py:125-388).
// B200 has no RT cores, so closest-hit queries are hand-written stack walks.
//
// The k-d walk (march.cuh) stays the frame kernel's default traversal; the
// LBVH serves region sets queried the reference's way — one closest-hit query
// per region visit — and exports the reference's node arrays.  Its answers are
// topology-independent (SURVEY.md §8(a) "BVH-independence"): slab parameters
// are monotone in the box bounds, the prune `lo_t > best_in` is strict and leaf
// ties resolve to the lower region id, so any valid BVH over the same active
// set gives the reference's (region, t_in, t_out) bit for bit.
#pragma once
#include "march.cuh"

namespace xb {

struct DevLbvh {
    int64_t n_prims = 0;
    int depth = 0;  // deepest leaf (root = 0)
    DevBuf<LbvhNode> nodes;
    DevBuf<int32_t> prims;
    double build_ms = 0.0;
    LbvhView view() const { return LbvhView{nodes.p, prims.p, n_prims}; }
};

// LBVH over the region ids prims_in[0, n) (device, any order)
void build_lbvh(const DevRegions& R, const int32_t* prims_in, int64_t n, DevLbvh& out, cudaStream_t s);

}  // namespace xb
