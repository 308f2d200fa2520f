// render.cuh — kernel parameter blocks for the march kernels.
#pragma once
#include "march.cuh"

namespace xb {

constexpr int kTileW = 16, kTileH = 8;  // screen tile; a warp owns an 8x4 quarter

// Passed by value as a __grid_constant__ kernel parameter (~8.6 KB < 32 KB):
// the call needs no device allocation, so concurrent renders are reentrant.
#ifndef XB_WALK_THREADS
#define XB_WALK_THREADS 128
#endif
constexpr int kWalkThreads = XB_WALK_THREADS;  // k_classify / k_walk / k_route / k_short block size
constexpr float kShortSamples = 24.f;  // short ray: complete list of <= kShortLeaves leaves, <= kShortSamples
constexpr int kShortLeaves = 8;        // estimated samples (RenderArgs.short_samples / short_leaves)
constexpr int kResume = 48;            // resume entries saved per truncated walk
// k_warp work statistics, compiled in only with `make DEBUG_CHUNKS=1` (the counters cost k_warp registers)
#ifndef XB_DEBUG_CHUNKS
#define XB_DEBUG_CHUNKS 0
#endif
constexpr bool kDebugChunks = XB_DEBUG_CHUNKS != 0;

struct RenderArgs {
    SceneView S;
    const uint8_t* vflags;  // per k-d node: subtree holds an active volume region
    const uint8_t* vmask4;  // per Kd4 node: active bit per child slot (k_warp)
    const uint8_t* imask4;  // same for the iso set
    // the active set k_classify / k_walk walk: the volume set, or the iso set in the iso phase
    const uint8_t* wflags;
    const uint8_t* wmask4;
    const float* wqmin;
    int walk_iso;
    const uint8_t* iflags;  // same for the iso predicate
    MarchConst M;
    int W, H;
    double pos[3], right[3], up[3], fwd[3];
    double tan_half, aspect;
    int tiles_x, tiles_y, tile_rank, tile_world, packed;
    uchar4* out8;
    double4* outf;
    int2* outcnt;
    unsigned long long* stats;  // [regions, samples, algorithmic bytes]
    unsigned long long* work_counter;  // k_frame / k_warp slot counter (zeroed per launch)
    int grab_div, grab_fixed;          // k_warp grab schedule (launch_render)
    int32_t* leaves;                   // k_walk -> k_warp: per slot leaf_cap region ids in ray order (or NULL)
    int32_t* leaf_count;               // per slot: count | 0x40000000 when truncated
    int leaf_cap;                      // list capacity per slot (k_walk2's cap)
    int walk_cap1;                     // k_walk's cap (pass 1)
    long long walk2_min;               // k_walk2 runs only for at least this many cap-cut walks
    int32_t* cut_list;                 // walks cut at walk_cap1 (k_walk2's work)
    int32_t* resume;                   // per slot: k_walk's ordered remainder when truncated (1 + 3 x kResume words)
    const float* vqmin;                // per region opacity minorant (k_walk early stop), may be NULL
    unsigned long long* walk_counter;  // list lengths: [0] short, [1] long, [2] cut, [3] hit, [4] any
    int32_t* hit_list;                 // candidate rays (k_walk's work), appended by k_classify
    int32_t* long_list;                // rays for k_warp / k_iso_warp (k_route, in hit-list order)
    int32_t* any_list;                 // long + short rays, merged (k_warp's work when k_short is off)
    unsigned long long* dbg;           // diagnostics (XB_DEBUG_CHUNKS): k_warp chunks, chunk lanes, rays, samples
    int fuse_short;                    // k_warp runs the short rays after the long ones (no k_short launch)
    unsigned long long* short_counter; // k_warp's short-ray grab counter
    int32_t* fixup_list;               // pixels for k_fixup (exact FP64 shading), or NULL
    unsigned long long* fixup_count;
    int cut_tau;                       // k_walk2 also continues walks stopped by the opacity minorant
    int32_t* blk_counts;               // k_walk -> k_route: short / long / cut rays per k_walk block
    int32_t* short_list;               // rays with a complete list of <= 8 leaves (k_short's work), or NULL
    long long short_min;               // k_short runs only for at least this many short rays (else k_warp takes them)
    int short_leaves;                  // short ray: complete list of <= short_leaves leaves ...
    float short_samples;               // ... and <= short_samples estimated samples
    float walk_tau_stop;               // k_walk stops listing once the opacity minorant passes this depth
    int use_lbvh;                      // tuning.traversal = 1: per-visit LBVH closest-hit queries (k_render)
    int kernel;                        // 0: walk pipeline + k_warp; 1: one thread per pixel (k_render)
    void* march_events;                // cudaEvent_t[2] recorded around the k_warp launch, or NULL
    LbvhView vlb, ilb;                 // LBVHs of the volume / iso active sets
    double* iso_tend;           // per slot: volume t_end (iso hit or clip end)
    double* iso_shade;          // per slot: headlight factor of the iso hit, < 0 when none
    double tf[1024];
};

struct RayBatchArgs {
    SceneView S;
    const uint8_t* vflags;
    const uint8_t* iflags;
    MarchConst M;
    int mode;  // 0 volume (integrate_ray), 1 iso (iso_intersect)
    int use_lbvh;
    LbvhView vlb, ilb;
    int64_t n;
    const double *o, *d, *t0, *t1, *rho;
    double* out;       // (n,4): RGBA, or (t_hit, gx, gy, gz)
    int64_t* counts;   // (n,2): regions, samples  | hit flag
    double tf[1024];
};

void launch_render(const RenderArgs& A, int64_t n_tiles_local, bool count, cudaStream_t s);
void launch_rays(const RayBatchArgs& B, cudaStream_t s);
void launch_unpack(const uchar4* packed, int64_t tiles_per_rank, int world, int tiles_x, int tiles_y, int W, int H,
                   uchar4* img, cudaStream_t s);

}  // namespace xb
