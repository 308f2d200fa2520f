/*
 * exabricks.h — C ABI of libexabricks.so, the B200-native (sm_100a) ExaBricks
 * hot path.  Plain pointers and sizes only; no torch / C++ types.
 *
 * The reference (`amrvol`, R/ = /root/reference/pkg/src/amrvol/) is Python +
 * numba with no FFI of its own; its operator boundary is the Python API plus
 * the numba kernel argument lists.  Each entry point below replaces one of
 * those (cited per function).  The Python package `paper_2009_03076_b200`
 * binds this header with ctypes and keeps the reference's Python signatures;
 * INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - return 0 on success, a negative XB_ERR_* code on failure; the message is
 *     available from xb_last_error() (thread-local);
 *   - host arrays are borrowed for the duration of the call;
 *   - objects (xb_model, xb_regions, xb_active) own device memory on the CUDA
 *     device they were created on and are immutable after creation, so any
 *     number of threads may render from them concurrently (the reference's
 *     service renders outside its lock, R/service.py:166-176);
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef EXABRICKS_H
#define EXABRICKS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library builds with -fvisibility=hidden */
#endif

#define XB_OK 0
#define XB_ERR_CUDA (-1)
#define XB_ERR_ARG (-2)
#define XB_ERR_INVALID_CELLS (-3) /* build_bricks input fails validate_cells */
#define XB_ERR_RANGE (-4)
#define XB_ERR_NO_TREE (-5)
#define XB_ERR_INTERNAL (-6)

typedef struct xb_cells xb_cells;     /* CellList on the device (R/model.py:124-205) */
typedef struct xb_model xb_model;     /* AmrModel on the device (R/model.py:250-343) */
typedef struct xb_regions xb_regions; /* RegionSet + its k-d tree (R/regions.py:35-79) */
typedef struct xb_active xb_active;   /* pruned region set = RegionBvh (R/accel.py:125-155) */

const char* xb_last_error(void);
int xb_abi_version(void);
int xb_device_count(int32_t* n);

/* ---- synthetic inputs: generate_synthetic(SyntheticSpec) R/io.py:198-295 ---- */
typedef struct {
    int32_t field;     /* 0 gaussian, 1 ramp, 2 constant, 3 octaves (make_field, R/io.py:221-235) */
    int32_t max_level;
    int64_t extent[3]; /* finest-cell units, multiples of 2**max_level */
    double threshold;  /* split when |grad f(centre)| * width >= threshold */
    int32_t n_holes, n_refine;
    double holes[32][4];  /* (cx, cy, cz, r): emitted cells with centre inside are dropped */
    double refine[32][4]; /* (cx, cy, cz, r): cells with centre inside always split */
    double center[3], sigma, amp;  /* GaussianField */
    double direction[3], offset;   /* RampField */
    double constant;               /* ConstantField */
    int32_t n_waves;               /* OctaveField: waves drawn on the host with the reference's RNG */
    double waves[8][5];            /* k[3], phase, amplitude */
} xb_synth_spec;

/* The cells stay on `device` (10^8-10^9 cells build without a host round trip). */
int xb_generate_synthetic(const xb_synth_spec* spec, int32_t device, xb_cells** out);
int xb_cells_info(const xb_cells* c, int64_t* n);
/* host arrays of length n: CellList.i/j/k/level (int32) and values (float32, one field) */
int xb_cells_download(const xb_cells* c, int32_t* i, int32_t* j, int32_t* k, int32_t* level, float* values);
void xb_cells_free(xb_cells* c);
/* streamed input (io.load_cells_device: .exacells read in chunks, R/io.py:88-113): allocate n cells on
 * `device`, then fill [offset, offset + count) from host or device arrays */
int xb_cells_create(int64_t n, int32_t device, xb_cells** out);
int xb_cells_upload(xb_cells* c, int64_t offset, int64_t count, const int32_t* i, const int32_t* j, const int32_t* k,
                    const int32_t* level, const float* values);
/* build_bricks on device-resident cells (same result as xb_build_bricks on the downloaded arrays) */
int xb_build_bricks_cells(const xb_cells* c, int32_t max_brick_width, int32_t keep_split_tree, xb_model** out);

/* ---- bricks: build_bricks(cells, BrickBuildParams) R/bricks.py:104-228 ---- */
/* values: (n, n_fields) row-major float32, as CellList.values (R/model.py:135-138); host or device pointers.
 * XB_ERR_INVALID_CELLS when validate_cells (R/model.py:392-457) would fail. */
int xb_build_bricks(const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* level, const float* values,
                    int64_t n, int32_t n_fields, int32_t max_brick_width, int32_t keep_split_tree, int32_t device,
                    xb_model** out);
/* AmrModel(field_names, brick_lower, brick_level, brick_dims, scalars) R/model.py:257-267; scalars (F, N). */
int xb_model_upload(const int32_t* lower, const int32_t* level, const int32_t* dims, const float* scalars,
                    int64_t n_bricks, int64_t n_cells, int32_t n_fields, int32_t device, xb_model** out);
int xb_model_info(const xb_model* m, int64_t* n_bricks, int64_t* n_cells, int32_t* n_fields, int64_t* n_tree_nodes);
int xb_model_download(const xb_model* m, int32_t* lower, int32_t* level, int32_t* dims, int64_t* offset,
                      float* scalars);
/* SplitTree arrays (R/bricks.py:45-68), preorder; only when built with keep_split_tree */
int xb_model_download_tree(const xb_model* m, int32_t* axis, double* pos, int32_t* left, int32_t* right,
                           int32_t* brick_start, int32_t* brick_count, double* box_lo, double* box_hi,
                           double* max_half);
/* attach SplitTree arrays (R/bricks.py:45-68) to a model, e.g. one created with xb_model_upload */
int xb_model_upload_tree(xb_model* m, int64_t n, const int32_t* axis, const double* pos, const int32_t* left,
                         const int32_t* right, const int32_t* brick_start, const int32_t* brick_count,
                         const double* box_lo, const double* box_hi, const double* max_half);
void xb_model_free(xb_model* m);

/* ---- regions: build_regions(model) R/regions.py:90-213 ---- */
int xb_build_regions(const xb_model* m, xb_regions** out);
int xb_regions_info(const xb_regions* r, int64_t* n_regions, int64_t* n_ids, int64_t* n_kd_nodes, int32_t* kd_depth);
/* value_range (R, F, 2) float64, finest_width (R) float64 — RegionSet layout */
int xb_regions_download(const xb_regions* r, double* lo, double* hi, int64_t* brick_off, int32_t* brick_ids,
                        double* value_range, double* finest_width);
void xb_regions_free(xb_regions* r);

/* ---- active sets: build_volume_bvh / build_iso_bvh / build_all_regions_bvh R/accel.py:227-247 ---- */
/* rgba: 256x4 float64 ramp (TransferFunction.rgba, R/accel.py:38-88) */
int xb_active_volume(const xb_regions* r, int32_t field, double tf_lo, double tf_hi, const double* rgba,
                     xb_active** out);
int xb_active_iso(const xb_regions* r, int32_t field, double iso_value, xb_active** out);
int xb_active_all(const xb_regions* r, xb_active** out);
int xb_active_info(const xb_active* a, int64_t* n_active, double* build_ms);
int xb_active_prims(const xb_active* a, int32_t* prims); /* ascending active region ids */
void xb_active_free(xb_active* a);

/* ---- render_frame R/render.py:654-691 (kernel body R/render.py:521-578) ---- */
typedef struct {
    int32_t width, height;
    double position[3];
    double right[3], up[3], forward[3]; /* Camera.basis(), R/render.py:73-79 */
    double tan_half;                    /* tan(radians(fov_y) / 2) */
    double aspect;                      /* width / height */
} xb_camera;

typedef struct {
    double samples_per_cell, rate_scale, early_term_threshold; /* MarchParams, R/render.py:92-116 */
    uint64_t seed;
    int32_t gradient_mode; /* GRADIENT_MODES: 0 none, 1 analytic, 2 central, 3 clampedCentral */
    int32_t n_planes;      /* clip planes (n, c): keep dot(n, x) <= c */
    double planes[6][4];
    int32_t iso_on;
    double iso_value;
    double iso_rgb[3]; /* ISO_COLOR, R/render.py:47 */
    double tf_lo, tf_hi;
    double tf_rgba[1024];
    int32_t use_tree; /* render_frame(use_celllocation=True): per-sample split-tree brick collection */
} xb_march;

/* Render the tiles of `tile_rank` out of `tile_world` (16x8-pixel tiles dealt
 * round-robin; world = 1 renders the frame).  rgba8: host or device; with
 * world == 1 it is the (H, W, 4) image, otherwise the rank's packed tiles
 * (xb_tile_count() tiles x 128 px x 4 B).  rgba_f64 / px_counts (int32
 * regions, samples per pixel): optional parity outputs, same layout, host or
 * device.  stats (may be NULL): [regions, samples, algorithmic bytes] (bytes
 * only when count_bytes != 0); a host pointer makes the call synchronous, a
 * device pointer (3 x int64) is filled on `stream` without host sync.  `vol`
 * may not be NULL; `iso` may. */
int xb_render(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* vol, const xb_active* iso,
              const xb_camera* cam, const xb_march* mp, int32_t tile_rank, int32_t tile_world, void* rgba8,
              double* rgba_f64, int32_t* px_counts, int64_t* stats, int32_t count_bytes, void* stream);
/* ---- frame-pipeline variants: A/B measurement and the parity matrix ----
 * Process-wide; xb_render / xb_integrate_rays take a snapshot when called.
 * The compiled defaults (xb_tuning_defaults) are the measured best
 * (DESIGN.md §5); nothing else — no environment variable — changes the
 * production path. */
typedef struct {
    int32_t kernel;     /* 0 (default): k_classify -> walk -> k_warp pipeline; 1: one thread per pixel (k_render) */
    int32_t traversal;  /* 0 (default): ordered k-d walk; 1: per-visit LBVH closest-hit queries, the
                           reference's traversal (R/accel.py:285-352; runs in the one-thread-per-pixel kernel) */
    int32_t walk_lists; /* 1 (default): k_walk leaf lists; 0: k_warp's warp frontier from the root only */
    int32_t leaf_cap;   /* 0 (default): two-pass walk (walk_cap1, then k_walk2 to 96); N > 0: one pass of N */
    int32_t walk_cap1;  /* pass-1 leaf cap of the two-pass walk (default 16; clamped to the list capacity) */
    int32_t short_rays; /* -1 (default): lane-per-ray phase when >= 1000 x SMs short rays; 0: never; 1: always */
    int64_t walk2_min;  /* k_walk2 runs when >= walk2_min walks were cut; -1 (default): 500 x SMs */
    int32_t fuse_short; /* 1 (default): short rays run inside k_warp after the long ones; 0: separate k_short */
    int32_t time_march; /* 1: record a CUDA event pair around every k_warp launch (xb_march_times); default 0 */
    int32_t short_leaves;  /* short ray: complete leaf list of <= short_leaves leaves (default 8) ... */
    int32_t short_samples; /* ... and <= short_samples estimated samples (default 24) */
    int32_t grab_div;      /* k_warp's guided ray grabs: remaining / (grab_div x warps), in [1, 32] (default 4) */
    int32_t grab_fixed;    /* > 0: fixed grabs of that many rays instead (default 0) */
} xb_tuning;
void xb_tuning_defaults(xb_tuning* t);
int xb_tuning_get(xb_tuning* t);
int xb_tuning_set(const xb_tuning* t); /* NULL restores the defaults */
/* Device time of the march kernel (k_warp, the frame's dominant kernel) of the
 * frames rendered with tuning.time_march = 1: waits for the recorded events and
 * returns up to `cap` elapsed times in ms, oldest first, in ms[0 .. *n); the
 * returned records are forgotten. */
int xb_march_times(double* ms, int32_t cap, int32_t* n);

int xb_tile_count(int32_t width, int32_t height, int32_t rank, int32_t world, int64_t* n_tiles, int32_t* tile_px);
/* gathered packed tiles (rank-major, tiles_per_rank each) -> (H, W, 4) image; device pointers */
int xb_unpack_tiles(const void* packed, int64_t tiles_per_rank, int32_t world, int32_t width, int32_t height,
                    void* rgba8, void* stream);

/* ---- single rays: integrate_ray R/render.py:613-632, iso_intersect 635-651 ---- */
/* host arrays; o, d (n,3) (d normalised by the caller), t0/t1/rho (n).
 * out (n,4) RGBA float64, counts (n,2) int64 regions/samples. */
int xb_integrate_rays(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* vol,
                      const xb_march* mp, int64_t n, const double* o, const double* d, const double* t0,
                      const double* t1, const double* rho, double* out, int64_t* counts);
/* out (n,4): t_hit, gx, gy, gz ; hit (n) */
int xb_iso_rays(const xb_model* m, const xb_regions* r, int32_t field, const xb_active* iso, const xb_march* mp,
                int64_t n, const double* o, const double* d, const double* t0, const double* t1, const double* rho,
                double* out, int32_t* hit);

/* ---- point reconstruction: basis_sample_region / gradient_analytic R/sampling.py:281-353 ---- */
/* region: per-point region id, or NULL to locate each point (point_to_region, R/regions.py:216-220).
 * acc (n, 9): num, den, [shifted num, dn(3), dd(3) when want_grad] (_gradient_bricks accumulators) */
int xb_sample_points(const xb_model* m, const xb_regions* r, int32_t field, int64_t n, const double* p,
                     const int32_t* region, int32_t want_grad, int32_t* region_out, double* acc);
/* basis_sample_oracle over the canonical cell order (R/sampling.py:291-298): out (n,2) num, den */
int xb_sample_scan(const xb_model* m, int32_t field, int64_t n, const double* p, double* out);
/* the same scan over any device cell list in its given order (basis_sample_oracle on a plain
 * CellList, R/sampling.py:291-298; one field, uploaded with xb_cells_create / xb_cells_upload) */
int xb_sample_scan_cells(const xb_cells* c, int64_t n, const double* p, double* out);
/* iterate_intervals R/accel.py:414-424 for n rays: up to cap intervals each (t_in, t_out, region), count */
int xb_trace_intervals(const xb_model* m, const xb_regions* r, const xb_active* a, int64_t n, const double* o,
                       const double* d, double t_start, double t_max, int32_t cap, double* t_in, double* t_out,
                       int32_t* region, int32_t* count);

/* ---- LBVH over an active set: RegionBvh (R/accel.py:125-224), _bvh_next_hit / _bvh_point_query (285-388) ----
 * Morton-sorted, Karras-built, refit on the GPU on first use.  Node arrays in
 * the reference's RegionBvh layout: 2n-1 nodes (internal, then one leaf per
 * region), f64 boxes (n,3), left/right (-1 at leaves), start (i64) / count
 * into prims; an empty set gives the reference's single dummy node. */
int xb_active_lbvh_info(const xb_active* a, int64_t* n_nodes, int32_t* depth, double* build_ms);
int xb_active_lbvh_download(const xb_active* a, double* node_lo, double* node_hi, int32_t* left, int32_t* right,
                            int64_t* start, int32_t* count, int32_t* prims);
/* iterate_intervals with one LBVH closest-hit query per region (the reference's traversal) */
int xb_trace_intervals_lbvh(const xb_model* m, const xb_regions* r, const xb_active* a, int64_t n, const double* o,
                            const double* d, double t_start, double t_max, int32_t cap, double* t_in, double* t_out,
                            int32_t* region, int32_t* count);
/* point_query (R/accel.py:408-411): active region whose half-open box holds p, else -1 */
int xb_point_query_lbvh(const xb_model* m, const xb_regions* r, const xb_active* a, int64_t n, const double* p,
                        int32_t* region);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* EXABRICKS_H */
