/*
 * xb_oracle.c — CPU restatement of the reference (`amrvol`, Python+numba)
 * algorithms on the ExaBricks hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * This file is the parity checker: `tests/`, `__graft_entry__.smoke()` and the
 * `cpu_baseline` / `--impl reference` legs of `bench.py` may load it; the
 * product path (`paper_2009_03076_b200`) never does.  Every function cites the
 * reference lines it restates (R/ = /root/reference/pkg/src/amrvol/).
 *
 * Parity: pinned against golden vectors produced by the reference itself
 * (tests/golden/make_golden.py) — builders bit-exact (np.array_equal on every
 * array), samples/gradients bit-exact, frames bit-exact in float64 RGBA.
 *
 * Floating point: compile with -ffp-contract=off and without -ffast-math so
 * every double op rounds once, like numba's LLVM code (no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define XO_API __attribute__((visibility("default")))

static inline int64_t floordiv64(int64_t a, int64_t b) { /* Python // for b > 0 */
    int64_t q = a / b;
    if ((a % b) != 0 && ((a < 0) != (b < 0))) q -= 1;
    return q;
}

/* ------------------------------------------------------------------------ */
/* growable arrays                                                          */

typedef struct { void* p; int64_t n, cap; size_t esz; } vec_t;
static void vec_init(vec_t* v, size_t esz) { v->p = NULL; v->n = 0; v->cap = 0; v->esz = esz; }
static void* vec_push(vec_t* v, int64_t k) {
    if (v->n + k > v->cap) {
        int64_t c = v->cap ? v->cap : 64;
        while (c < v->n + k) c *= 2;
        v->p = realloc(v->p, (size_t)c * v->esz);
        v->cap = c;
    }
    void* out = (char*)v->p + (size_t)v->n * v->esz;
    v->n += k;
    return out;
}

/* ======================================================================== */
/* build_bricks  (R/bricks.py:104-228)                                      */

typedef struct {
    int64_t n_bricks, n_cells, n_fields, n_nodes;
    int32_t *lower, *level, *dims; /* (B,3) (B) (B,3) */
    int64_t *offset;               /* B+1 */
    float* scalars;                /* (F, N) */
    /* split tree, preorder (R/bricks.py:45-101) */
    int32_t *t_axis, *t_left, *t_right, *t_bstart, *t_bcount;
    double *t_pos, *t_lo, *t_hi, *t_mh;
} xo_bricks_t;

typedef struct {
    const int64_t *ci, *cj, *ck, *clev; /* sorted */
    const float* cvals;                 /* (n, F) sorted rows */
    int64_t F, maxw;
    int64_t* tmp;
    vec_t lower, level, dims, slabs_off, slab_vals; /* slab_vals: per brick F*cnt floats, field-major */
    int keep_tree;
    vec_t axis, pos, left, right, bstart, bcount, blo, bhi, mh;
} bb_ctx;

static int64_t bb_emit(bb_ctx* c, const int64_t* idx, int64_t cnt, const int64_t lo[3], int64_t level, const int64_t dims[3]) {
    /* emit_brick, R/bricks.py:135-147 */
    int64_t nx = dims[0], ny = dims[1], nz = dims[2], ncell = nx * ny * nz;
    int32_t* L = vec_push(&c->lower, 3);
    L[0] = (int32_t)lo[0]; L[1] = (int32_t)lo[1]; L[2] = (int32_t)lo[2];
    *(int32_t*)vec_push(&c->level, 1) = (int32_t)level;
    int32_t* D = vec_push(&c->dims, 3);
    D[0] = (int32_t)nx; D[1] = (int32_t)ny; D[2] = (int32_t)nz;
    *(int64_t*)vec_push(&c->slabs_off, 1) = c->slab_vals.n;
    float* slab = vec_push(&c->slab_vals, c->F * ncell);
    for (int64_t t = 0; t < cnt; t++) {
        int64_t q = idx[t];
        int64_t gx = (c->ci[q] - lo[0]) >> level;
        int64_t gy = (c->cj[q] - lo[1]) >> level;
        int64_t gz = (c->ck[q] - lo[2]) >> level;
        int64_t slot = gx + nx * (gy + ny * gz);
        for (int64_t f = 0; f < c->F; f++) slab[f * ncell + slot] = c->cvals[q * c->F + f];
    }
    return c->level.n - 1;
}

static int64_t bb_tree_add(bb_ctx* c) {
    if (!c->keep_tree) return -1;
    *(int32_t*)vec_push(&c->axis, 1) = 0;
    *(double*)vec_push(&c->pos, 1) = 0.0;
    *(int32_t*)vec_push(&c->left, 1) = 0;
    *(int32_t*)vec_push(&c->right, 1) = 0;
    *(int32_t*)vec_push(&c->bstart, 1) = 0;
    *(int32_t*)vec_push(&c->bcount, 1) = 0;
    double* a = vec_push(&c->blo, 3); a[0] = a[1] = a[2] = 0.0;
    double* b = vec_push(&c->bhi, 3); b[0] = b[1] = b[2] = 0.0;
    *(double*)vec_push(&c->mh, 1) = 0.0;
    return c->axis.n - 1;
}

#define TREE_I32(vec, node) (((int32_t*)(c->vec).p)[node])
#define TREE_F64(vec, node) (((double*)(c->vec).p)[node])

/* build(idx), R/bricks.py:155-212; idx is a window of c->tmp-permutable ids */
static int64_t bb_build(bb_ctx* c, int64_t* idx, int64_t cnt) {
    int64_t lo[3] = {INT64_MAX, INT64_MAX, INT64_MAX}, hi[3] = {INT64_MIN, INT64_MIN, INT64_MIN};
    int64_t lmin = INT64_MAX, lmax = INT64_MIN;
    for (int64_t t = 0; t < cnt; t++) { /* node_box, R/bricks.py:149-153 */
        int64_t q = idx[t], w = (int64_t)1 << c->clev[q];
        int64_t co[3] = {c->ci[q], c->cj[q], c->ck[q]};
        for (int a = 0; a < 3; a++) {
            if (co[a] < lo[a]) lo[a] = co[a];
            if (co[a] + w > hi[a]) hi[a] = co[a] + w;
        }
        if (c->clev[q] < lmin) lmin = c->clev[q];
        if (c->clev[q] > lmax) lmax = c->clev[q];
    }
    int64_t ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    int64_t node = bb_tree_add(c);
    if (node >= 0) {
        for (int a = 0; a < 3; a++) {
            ((double*)c->blo.p)[node * 3 + a] = (double)lo[a];
            ((double*)c->bhi.p)[node * 3 + a] = (double)hi[a];
        }
        TREE_F64(mh, node) = 0.5 * ldexp(1.0, (int)lmax);
    }
    int64_t w = (int64_t)1 << lmax;
    __int128 vol = (__int128)ext[0] * ext[1] * ext[2];
    __int128 need = (__int128)cnt * w * w * w;
    int filled = (lmin == lmax) && need == vol; /* R/bricks.py:167 */
    int64_t dims[3] = {ext[0] >> lmax, ext[1] >> lmax, ext[2] >> lmax};
    int fits = dims[0] <= c->maxw && dims[1] <= c->maxw && dims[2] <= c->maxw;
    if (filled && fits) {
        int64_t b = bb_emit(c, idx, cnt, lo, lmax, dims);
        if (node >= 0) { TREE_I32(axis, node) = -1; TREE_I32(bstart, node) = (int32_t)b; TREE_I32(bcount, node) = 1; }
        return node;
    }
    int axis = 0; /* argmax, first max: R/bricks.py:179 */
    if (ext[1] > ext[axis]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    int64_t wc = w, a_lo = lo[axis], a_hi = hi[axis];
    int64_t mid2 = a_lo + a_hi;
    int64_t plane = floordiv64(mid2 + wc, 2 * wc) * wc; /* R/bricks.py:183 */
    if (!(a_lo < plane && plane < a_hi)) {
        int64_t k_lo = floordiv64(a_lo, wc) + 1;
        int64_t k_hi = floordiv64(a_hi - 1, wc);
        if (k_lo > k_hi) { /* per-cell leaves, R/bricks.py:187-200 */
            int64_t first = -1;
            for (int64_t t = 0; t < cnt; t++) {
                int64_t q = idx[t];
                int64_t clo[3] = {c->ci[q], c->cj[q], c->ck[q]}, one[3] = {1, 1, 1};
                int64_t b = bb_emit(c, &idx[t], 1, clo, c->clev[q], one);
                if (first < 0) first = b;
            }
            if (node >= 0) { TREE_I32(axis, node) = -1; TREE_I32(bstart, node) = (int32_t)first; TREE_I32(bcount, node) = (int32_t)cnt; }
            return node;
        }
        int64_t k_mid = floordiv64(mid2 + wc, 2 * wc);
        if (k_mid < k_lo) k_mid = k_lo;
        if (k_mid > k_hi) k_mid = k_hi;
        plane = k_mid * wc;
    }
    /* stable partition: left = coord[axis] < plane (R/bricks.py:204) */
    int64_t nl = 0, nr = 0;
    int64_t* tmp = c->tmp;
    const int64_t* co = axis == 0 ? c->ci : (axis == 1 ? c->cj : c->ck);
    for (int64_t t = 0; t < cnt; t++) if (co[idx[t]] < plane) idx[nl++] = idx[t]; else tmp[nr++] = idx[t];
    memcpy(idx + nl, tmp, (size_t)nr * sizeof(int64_t));
    int64_t l = bb_build(c, idx, nl);
    int64_t r = bb_build(c, idx + nl, nr);
    if (node >= 0) {
        TREE_I32(axis, node) = axis;
        TREE_F64(pos, node) = (double)plane;
        TREE_I32(left, node) = (int32_t)l;
        TREE_I32(right, node) = (int32_t)r;
    }
    return node;
}

/* lexsort by (level, k, j, i), R/bricks.py:120 */
static const int32_t *srt_i, *srt_j, *srt_k, *srt_l;
static int cell_cmp(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    if (srt_l[x] != srt_l[y]) return srt_l[x] < srt_l[y] ? -1 : 1;
    if (srt_k[x] != srt_k[y]) return srt_k[x] < srt_k[y] ? -1 : 1;
    if (srt_j[x] != srt_j[y]) return srt_j[x] < srt_j[y] ? -1 : 1;
    if (srt_i[x] != srt_i[y]) return srt_i[x] < srt_i[y] ? -1 : 1;
    return x < y ? -1 : (x > y); /* lexsort is stable */
}

/* The same stable lexsort as an LSD radix sort on packed (level, k, j, i)
 * keys (offset by their minima) when they fit in 64 bits: equal keys keep
 * their input order, like np.lexsort.  Returns 0 when they do not fit. */
static int bits_for(int64_t range) { int b = 0; while (b < 63 && ((int64_t)1 << b) <= range) b++; return b; }
static int radix_lexsort(int64_t n, const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* lev,
                         int64_t* order) {
    if (n < 2) return 1;
    int64_t mn[4], mx[4];
    const int32_t* a[4] = {i, j, k, lev};
    for (int c = 0; c < 4; c++) {
        mn[c] = INT64_MAX; mx[c] = INT64_MIN;
        for (int64_t t = 0; t < n; t++) { if (a[c][t] < mn[c]) mn[c] = a[c][t]; if (a[c][t] > mx[c]) mx[c] = a[c][t]; }
    }
    int b[4], tot = 0;
    for (int c = 0; c < 4; c++) { b[c] = bits_for(mx[c] - mn[c]); tot += b[c]; }
    if (tot > 64) return 0;
    uint64_t* key = malloc(sizeof(uint64_t) * n);
    uint64_t* key2 = malloc(sizeof(uint64_t) * n);
    int64_t* ord2 = malloc(sizeof(int64_t) * n);
    for (int64_t t = 0; t < n; t++) {  /* i lowest, level highest */
        uint64_t v = 0; int sh = 0;
        for (int c = 0; c < 4; c++) { v |= (uint64_t)(a[c][t] - mn[c]) << sh; sh += b[c]; }
        key[t] = v;
    }
    int64_t cnt[65536];
    for (int pass = 0; pass * 16 < tot; pass++) {
        int sh = pass * 16;
        memset(cnt, 0, sizeof cnt);
        for (int64_t t = 0; t < n; t++) cnt[(key[t] >> sh) & 0xffff]++;
        int64_t sum = 0;
        for (int d = 0; d < 65536; d++) { int64_t c = cnt[d]; cnt[d] = sum; sum += c; }
        for (int64_t t = 0; t < n; t++) {
            int64_t p = cnt[(key[t] >> sh) & 0xffff]++;
            key2[p] = key[t];
            ord2[p] = order[t];
        }
        uint64_t* tk = key; key = key2; key2 = tk;
        memcpy(order, ord2, sizeof(int64_t) * n);
    }
    free(key); free(key2); free(ord2);
    return 1;
}

XO_API xo_bricks_t* xo_build_bricks(int64_t n, const int32_t* i, const int32_t* j, const int32_t* k, const int32_t* lev,
                                    const float* vals, int64_t F, int64_t maxw, int keep_tree) {
    xo_bricks_t* out = calloc(1, sizeof(xo_bricks_t));
    out->n_fields = F;
    int64_t* order = malloc(sizeof(int64_t) * (n ? n : 1));
    for (int64_t t = 0; t < n; t++) order[t] = t;
    if (!radix_lexsort(n, i, j, k, lev, order)) {
        srt_i = i; srt_j = j; srt_k = k; srt_l = lev;
        qsort(order, (size_t)n, sizeof(int64_t), cell_cmp);
    }
    int64_t *ci = malloc(8 * (n + 1)), *cj = malloc(8 * (n + 1)), *ck = malloc(8 * (n + 1)), *cl = malloc(8 * (n + 1));
    float* cv = malloc(sizeof(float) * (n * F + 1));
    for (int64_t t = 0; t < n; t++) {
        int64_t q = order[t];
        ci[t] = i[q]; cj[t] = j[q]; ck[t] = k[q]; cl[t] = lev[q];
        for (int64_t f = 0; f < F; f++) cv[t * F + f] = vals[q * F + f];
    }
    bb_ctx c;
    memset(&c, 0, sizeof(c));
    c.ci = ci; c.cj = cj; c.ck = ck; c.clev = cl; c.cvals = cv; c.F = F; c.maxw = maxw; c.keep_tree = keep_tree;
    c.tmp = malloc(8 * (n + 1));
    vec_init(&c.lower, 4); vec_init(&c.level, 4); vec_init(&c.dims, 4); vec_init(&c.slabs_off, 8); vec_init(&c.slab_vals, 4);
    vec_init(&c.axis, 4); vec_init(&c.pos, 8); vec_init(&c.left, 4); vec_init(&c.right, 4); vec_init(&c.bstart, 4);
    vec_init(&c.bcount, 4); vec_init(&c.blo, 8); vec_init(&c.bhi, 8); vec_init(&c.mh, 8);
    int64_t* idx = malloc(8 * (n + 1));
    for (int64_t t = 0; t < n; t++) idx[t] = t;
    if (n > 0) bb_build(&c, idx, n);
    int64_t B = c.level.n;
    out->n_bricks = B;
    out->lower = c.lower.p; out->level = c.level.p; out->dims = c.dims.p;
    out->offset = malloc(8 * (B + 1));
    out->offset[0] = 0;
    for (int64_t b = 0; b < B; b++) out->offset[b + 1] = out->offset[b] + (int64_t)out->dims[3 * b] * out->dims[3 * b + 1] * out->dims[3 * b + 2];
    int64_t N = out->offset[B];
    out->n_cells = N;
    out->scalars = malloc(sizeof(float) * (F * N + 1));
    for (int64_t b = 0; b < B; b++) {
        int64_t cnt = out->offset[b + 1] - out->offset[b];
        const float* slab = (const float*)c.slab_vals.p + ((int64_t*)c.slabs_off.p)[b];
        for (int64_t f = 0; f < F; f++) memcpy(out->scalars + f * N + out->offset[b], slab + f * cnt, sizeof(float) * cnt);
    }
    out->n_nodes = keep_tree ? c.axis.n : 0;
    out->t_axis = c.axis.p; out->t_pos = c.pos.p; out->t_left = c.left.p; out->t_right = c.right.p;
    out->t_bstart = c.bstart.p; out->t_bcount = c.bcount.p; out->t_lo = c.blo.p; out->t_hi = c.bhi.p; out->t_mh = c.mh.p;
    free(c.slabs_off.p); free(c.slab_vals.p); free(c.tmp); free(idx);
    free(order); free(ci); free(cj); free(ck); free(cl); free(cv);
    return out;
}

XO_API void xo_bricks_free(xo_bricks_t* b) {
    if (!b) return;
    free(b->lower); free(b->level); free(b->dims); free(b->offset); free(b->scalars);
    free(b->t_axis); free(b->t_pos); free(b->t_left); free(b->t_right); free(b->t_bstart); free(b->t_bcount);
    free(b->t_lo); free(b->t_hi); free(b->t_mh);
    free(b);
}

/* ======================================================================== */
/* build_regions  (R/regions.py:82-213)                                     */

typedef struct {
    int64_t n_regions, n_ids, n_fields;
    double *lo, *hi;      /* (R,3) */
    int64_t* brick_off;   /* R+1 */
    int32_t* brick_ids;
    double* value_range;  /* (R,F,2) */
    double* finest;       /* R */
    /* k-d split record of the build, preorder (for diagnostics) */
} xo_regions_t;

typedef struct { int64_t lo[3], hi[3]; int64_t n; int64_t* flo; int64_t* fhi; int32_t* fid; } rg_node;

XO_API xo_regions_t* xo_build_regions(int64_t B, const int32_t* lower, const int32_t* level, const int32_t* dims,
                                      const int64_t* boffset, const float* scalars, int64_t F, int64_t N) {
    xo_regions_t* out = calloc(1, sizeof(xo_regions_t));
    out->n_fields = F;
    if (B == 0) {
        out->brick_off = calloc(1, 8);
        return out;
    }
    /* _support_boxes_halfunits, R/regions.py:82-87 */
    rg_node root;
    root.n = B;
    root.flo = malloc(8 * 3 * B); root.fhi = malloc(8 * 3 * B); root.fid = malloc(4 * B);
    for (int a = 0; a < 3; a++) { root.lo[a] = INT64_MAX; root.hi[a] = INT64_MIN; }
    for (int64_t b = 0; b < B; b++) {
        int64_t w = (int64_t)1 << level[b];
        for (int a = 0; a < 3; a++) {
            int64_t lo = lower[3 * b + a], hi = lo + (int64_t)dims[3 * b + a] * w;
            root.flo[3 * b + a] = 2 * lo - w;
            root.fhi[3 * b + a] = 2 * hi + w;
            if (root.flo[3 * b + a] < root.lo[a]) root.lo[a] = root.flo[3 * b + a];
            if (root.fhi[3 * b + a] > root.hi[a]) root.hi[a] = root.fhi[3 * b + a];
        }
        root.fid[b] = (int32_t)b;
    }
    vec_t stack, leaf_lo, leaf_hi, leaf_off, leaf_ids;
    vec_init(&stack, sizeof(rg_node)); vec_init(&leaf_lo, 8); vec_init(&leaf_hi, 8); vec_init(&leaf_off, 8); vec_init(&leaf_ids, 4);
    *(int64_t*)vec_push(&leaf_off, 1) = 0;
    *(rg_node*)vec_push(&stack, 1) = root;
    while (stack.n > 0) { /* R/regions.py:115-149 */
        rg_node nd = ((rg_node*)stack.p)[--stack.n];
        int64_t wdt[3] = {nd.hi[0] - nd.lo[0], nd.hi[1] - nd.lo[1], nd.hi[2] - nd.lo[2]};
        int ord[3] = {0, 1, 2}; /* stable argsort of -width */
        for (int x = 1; x < 3; x++)
            for (int y = x; y > 0 && wdt[ord[y]] > wdt[ord[y - 1]]; y--) { int t = ord[y]; ord[y] = ord[y - 1]; ord[y - 1] = t; }
        int axis = -1;
        int64_t plane = 0;
        for (int oi = 0; oi < 3 && axis < 0; oi++) {
            int a = ord[oi];
            int64_t best_d = INT64_MAX, best_f = 0;
            int found = 0;
            for (int64_t t = 0; t < nd.n; t++) {
                int64_t faces[2] = {nd.flo[3 * t + a], nd.fhi[3 * t + a]};
                for (int s = 0; s < 2; s++) {
                    int64_t f = faces[s];
                    if (f > nd.lo[a] && f < nd.hi[a]) {
                        int64_t d = 2 * f - (nd.lo[a] + nd.hi[a]);
                        if (d < 0) d = -d;
                        if (!found || d < best_d || (d == best_d && f < best_f)) { best_d = d; best_f = f; found = 1; }
                    }
                }
            }
            if (found) { axis = a; plane = best_f; }
        }
        if (axis < 0) {
            if (nd.n > 0) { /* fid stays ascending under the stable splits: np.sort is the identity */
                int64_t* L = vec_push(&leaf_lo, 3); int64_t* H = vec_push(&leaf_hi, 3);
                for (int a = 0; a < 3; a++) { L[a] = nd.lo[a]; H[a] = nd.hi[a]; }
                int32_t* ids = vec_push(&leaf_ids, nd.n);
                memcpy(ids, nd.fid, 4 * nd.n);
                /* insertion sort for safety (np.sort) */
                for (int64_t x = 1; x < nd.n; x++)
                    for (int64_t y = x; y > 0 && ids[y] < ids[y - 1]; y--) { int32_t t = ids[y]; ids[y] = ids[y - 1]; ids[y - 1] = t; }
                *(int64_t*)vec_push(&leaf_off, 1) = leaf_ids.n;
            }
            free(nd.flo); free(nd.fhi); free(nd.fid);
            continue;
        }
        int64_t nl = 0, nr = 0;
        for (int64_t t = 0; t < nd.n; t++) { nl += nd.flo[3 * t + axis] < plane; nr += nd.fhi[3 * t + axis] > plane; }
        rg_node L, Rn;
        L.n = nl; Rn.n = nr;
        L.flo = malloc(8 * 3 * (nl + 1)); L.fhi = malloc(8 * 3 * (nl + 1)); L.fid = malloc(4 * (nl + 1));
        Rn.flo = malloc(8 * 3 * (nr + 1)); Rn.fhi = malloc(8 * 3 * (nr + 1)); Rn.fid = malloc(4 * (nr + 1));
        int64_t il = 0, ir = 0;
        for (int64_t t = 0; t < nd.n; t++) {
            if (nd.flo[3 * t + axis] < plane) {
                memcpy(&L.flo[3 * il], &nd.flo[3 * t], 24); memcpy(&L.fhi[3 * il], &nd.fhi[3 * t], 24);
                if (L.fhi[3 * il + axis] > plane) L.fhi[3 * il + axis] = plane;
                L.fid[il++] = nd.fid[t];
            }
            if (nd.fhi[3 * t + axis] > plane) {
                memcpy(&Rn.flo[3 * ir], &nd.flo[3 * t], 24); memcpy(&Rn.fhi[3 * ir], &nd.fhi[3 * t], 24);
                if (Rn.flo[3 * ir + axis] < plane) Rn.flo[3 * ir + axis] = plane;
                Rn.fid[ir++] = nd.fid[t];
            }
        }
        for (int a = 0; a < 3; a++) { L.lo[a] = nd.lo[a]; L.hi[a] = nd.hi[a]; Rn.lo[a] = nd.lo[a]; Rn.hi[a] = nd.hi[a]; }
        L.hi[axis] = plane;
        Rn.lo[axis] = plane;
        free(nd.flo); free(nd.fhi); free(nd.fid);
        *(rg_node*)vec_push(&stack, 1) = Rn; /* right first: left processed first */
        *(rg_node*)vec_push(&stack, 1) = L;
    }
    free(stack.p);
    int64_t R = leaf_lo.n / 3;
    out->n_regions = R;
    out->n_ids = leaf_ids.n;
    out->brick_off = leaf_off.p;
    out->brick_ids = leaf_ids.p;
    out->lo = malloc(8 * 3 * (R + 1)); out->hi = malloc(8 * 3 * (R + 1));
    int64_t* lh = leaf_lo.p; int64_t* hh = leaf_hi.p;
    for (int64_t t = 0; t < 3 * R; t++) { out->lo[t] = (double)lh[t] / 2.0; out->hi[t] = (double)hh[t] / 2.0; }
    out->value_range = malloc(8 * (R * F * 2 + 1));
    out->finest = malloc(8 * (R + 1));
    /* _region_metadata, R/regions.py:174-213 */
    for (int64_t r = 0; r < R; r++) {
        for (int64_t f = 0; f < F; f++) { out->value_range[(r * F + f) * 2] = INFINITY; out->value_range[(r * F + f) * 2 + 1] = -INFINITY; }
        double finest = INFINITY;
        for (int64_t t = out->brick_off[r]; t < out->brick_off[r + 1]; t++) {
            int64_t b = out->brick_ids[t];
            int64_t lev = level[b];
            int64_t w_h = (int64_t)2 << lev, half_h = (int64_t)1 << lev;
            double w_world = ldexp(1.0, (int)lev);
            if (w_world < finest) finest = w_world;
            int64_t n3[3] = {dims[3 * b], dims[3 * b + 1], dims[3 * b + 2]};
            int64_t i0[3], i1[3];
            for (int a = 0; a < 3; a++) {
                int64_t blh = 2 * (int64_t)lower[3 * b + a];
                int64_t x0 = floordiv64(lh[3 * r + a] - blh - half_h, w_h);
                int64_t x1 = floordiv64(hh[3 * r + a] - blh + half_h - 1, w_h);
                i0[a] = x0 > 0 ? x0 : 0;
                i1[a] = x1 < n3[a] - 1 ? x1 : n3[a] - 1;
            }
            int64_t base = boffset[b];
            for (int64_t z = i0[2]; z <= i1[2]; z++)
                for (int64_t y = i0[1]; y <= i1[1]; y++) {
                    int64_t row = base + n3[0] * (y + n3[1] * z);
                    for (int64_t x = i0[0]; x <= i1[0]; x++)
                        for (int64_t f = 0; f < F; f++) {
                            double v = scalars[f * N + row + x];
                            double* vr = &out->value_range[(r * F + f) * 2];
                            if (v < vr[0]) vr[0] = v;
                            if (v > vr[1]) vr[1] = v;
                        }
                }
        }
        out->finest[r] = finest;
    }
    free(leaf_lo.p); free(leaf_hi.p);
    return out;
}

XO_API void xo_regions_free(xo_regions_t* r) {
    if (!r) return;
    free(r->lo); free(r->hi); free(r->brick_off); free(r->brick_ids); free(r->value_range); free(r->finest);
    free(r);
}

/* ======================================================================== */
/* transfer function  (R/accel.py:56-115, R/render.py:236-254)              */

XO_API double xo_max_opacity(double lo, double hi, const double* rgba, double vmin, double vmax) {
    double scale = 255.0 / (hi - lo);
    double x0 = (vmin - lo) * scale, x1 = (vmax - lo) * scale;
    x0 = x0 < 0.0 ? 0.0 : x0; x0 = x0 > 255.0 ? 255.0 : x0;
    x1 = x1 < 0.0 ? 0.0 : x1; x1 = x1 > 255.0 ? 255.0 : x1;
    double m = -INFINITY;
    double xs[2] = {x0, x1};
    for (int s = 0; s < 2; s++) {
        double x = xs[s];
        int64_t i = (int64_t)x;
        double v;
        if (i >= 255) v = rgba[255 * 4 + 3];
        else { double f = x - (double)i; v = (1.0 - f) * rgba[i * 4 + 3] + f * rgba[(i + 1) * 4 + 3]; }
        if (s == 0 || v > m) m = v;
    }
    int64_t k0 = (int64_t)ceil(x0), k1 = (int64_t)floor(x1);
    for (int64_t k = k0; k <= k1; k++) if (rgba[k * 4 + 3] > m) m = rgba[k * 4 + 3];
    return m;
}

/* the volume active set over every region (build_volume_bvh's filter, R/accel.py:227-234):
 * ids with max_opacity(tf, vr[r]) > 0, ascending; returns their count */
XO_API int64_t xo_active_volume(double lo, double hi, const double* rgba, int64_t n, const double* vr, int64_t stride,
                                int64_t* out) {
    int64_t k = 0;
    for (int64_t r = 0; r < n; r++)
        if (xo_max_opacity(lo, hi, rgba, vr[r * stride], vr[r * stride + 1]) > 0.0) out[k++] = r;
    return k;
}

static inline void tf_eval(double tf_lo, double tf_hi, const double* rgba, double v, double out[4]) {
    double t = (v - tf_lo) / (tf_hi - tf_lo);
    if (t < 0.0) t = 0.0;
    else if (t > 1.0) t = 1.0;
    double x = t * 255.0;
    int64_t i = (int64_t)x;
    if (i >= 255) { for (int c = 0; c < 4; c++) out[c] = rgba[255 * 4 + c]; return; }
    double f = x - (double)i, g = 1.0 - f;
    for (int c = 0; c < 4; c++) out[c] = g * rgba[i * 4 + c] + f * rgba[(i + 1) * 4 + c];
}

/* ======================================================================== */
/* BVH (R/accel.py:161-388)                                                 */

typedef struct {
    int64_t n_nodes, n_prims;
    double *nlo, *nhi;
    int32_t *left, *right, *count, *prims;
    int64_t* start;
} xo_bvh_t;

typedef struct { const double *lo, *hi, *cen; const int64_t* active; vec_t nlo, nhi, l, r, s, c, prims; int64_t* tmp; } bvh_ctx;

static int bvh_axis_key;
static const double* bvh_cen_sort;
static const int64_t* bvh_act_sort;
static int bvh_cmp(const void* a, const void* b) { /* lexsort((active[sel], c[:,axis])) */
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    double cx = bvh_cen_sort[3 * x + bvh_axis_key], cy = bvh_cen_sort[3 * y + bvh_axis_key];
    if (cx < cy) return -1;
    if (cx > cy) return 1;
    if (bvh_act_sort[x] != bvh_act_sort[y]) return bvh_act_sort[x] < bvh_act_sort[y] ? -1 : 1;
    return x < y ? -1 : (x > y);
}

static int64_t bvh_rec(bvh_ctx* c, int64_t* sel, int64_t n) {
    int64_t node = c->l.n;
    double* lo = vec_push(&c->nlo, 3); double* hi = vec_push(&c->nhi, 3);
    for (int a = 0; a < 3; a++) { lo[a] = INFINITY; hi[a] = -INFINITY; }
    for (int64_t t = 0; t < n; t++)
        for (int a = 0; a < 3; a++) {
            double v = c->lo[3 * sel[t] + a], w = c->hi[3 * sel[t] + a];
            if (v < ((double*)c->nlo.p)[3 * node + a]) ((double*)c->nlo.p)[3 * node + a] = v;
            if (w > ((double*)c->nhi.p)[3 * node + a]) ((double*)c->nhi.p)[3 * node + a] = w;
        }
    *(int32_t*)vec_push(&c->l, 1) = -1; *(int32_t*)vec_push(&c->r, 1) = -1;
    *(int64_t*)vec_push(&c->s, 1) = 0; *(int32_t*)vec_push(&c->c, 1) = 0;
    if (n <= 4) {
        ((int64_t*)c->s.p)[node] = c->prims.n;
        ((int32_t*)c->c.p)[node] = (int32_t)n;
        for (int64_t t = 0; t < n; t++) *(int32_t*)vec_push(&c->prims, 1) = (int32_t)c->active[sel[t]];
        return node;
    }
    double mx[3] = {-INFINITY, -INFINITY, -INFINITY}, mn[3] = {INFINITY, INFINITY, INFINITY};
    for (int64_t t = 0; t < n; t++)
        for (int a = 0; a < 3; a++) {
            double v = c->cen[3 * sel[t] + a];
            if (v > mx[a]) mx[a] = v;
            if (v < mn[a]) mn[a] = v;
        }
    int axis = 0;
    double best = mx[0] - mn[0];
    for (int a = 1; a < 3; a++) if (mx[a] - mn[a] > best) { best = mx[a] - mn[a]; axis = a; }
    bvh_axis_key = axis; bvh_cen_sort = c->cen; bvh_act_sort = c->active;
    qsort(sel, (size_t)n, sizeof(int64_t), bvh_cmp);
    int64_t half = n / 2;
    int64_t l = bvh_rec(c, sel, half);
    int64_t r = bvh_rec(c, sel + half, n - half);
    ((int32_t*)c->l.p)[node] = (int32_t)l;
    ((int32_t*)c->r.p)[node] = (int32_t)r;
    return node;
}

XO_API xo_bvh_t* xo_build_bvh(int64_t n_active, const int64_t* active, const double* region_lo, const double* region_hi) {
    bvh_ctx c;
    memset(&c, 0, sizeof(c));
    vec_init(&c.nlo, 8); vec_init(&c.nhi, 8); vec_init(&c.l, 4); vec_init(&c.r, 4); vec_init(&c.s, 8); vec_init(&c.c, 4); vec_init(&c.prims, 4);
    double* lo = malloc(8 * 3 * (n_active + 1));
    double* hi = malloc(8 * 3 * (n_active + 1));
    double* cen = malloc(8 * 3 * (n_active + 1));
    for (int64_t t = 0; t < n_active; t++)
        for (int a = 0; a < 3; a++) {
            lo[3 * t + a] = region_lo[3 * active[t] + a];
            hi[3 * t + a] = region_hi[3 * active[t] + a];
            cen[3 * t + a] = 0.5 * (lo[3 * t + a] + hi[3 * t + a]);
        }
    c.lo = lo; c.hi = hi; c.cen = cen; c.active = active;
    int64_t* sel = malloc(8 * (n_active + 1));
    for (int64_t t = 0; t < n_active; t++) sel[t] = t;
    if (n_active) bvh_rec(&c, sel, n_active);
    else {
        double* a = vec_push(&c.nlo, 3); double* b = vec_push(&c.nhi, 3);
        for (int x = 0; x < 3; x++) { a[x] = INFINITY; b[x] = -INFINITY; }
        *(int32_t*)vec_push(&c.l, 1) = -1; *(int32_t*)vec_push(&c.r, 1) = -1;
        *(int64_t*)vec_push(&c.s, 1) = 0; *(int32_t*)vec_push(&c.c, 1) = 0;
    }
    xo_bvh_t* out = calloc(1, sizeof(xo_bvh_t));
    out->n_nodes = c.l.n; out->n_prims = c.prims.n;
    out->nlo = c.nlo.p; out->nhi = c.nhi.p; out->left = c.l.p; out->right = c.r.p; out->start = c.s.p; out->count = c.c.p;
    out->prims = c.prims.p ? c.prims.p : calloc(1, 4);
    free(lo); free(hi); free(cen); free(sel);
    return out;
}

XO_API void xo_bvh_free(xo_bvh_t* b) {
    if (!b) return;
    free(b->nlo); free(b->nhi); free(b->left); free(b->right); free(b->start); free(b->count); free(b->prims);
    free(b);
}

static inline void slab(const double* lo, const double* hi, const double o[3], const double d[3], double* tmin_o, double* tmax_o) {
    /* _slab, R/accel.py:254-282 */
    double tmin = -INFINITY, tmax = INFINITY;
    for (int a = 0; a < 3; a++) {
        if (d[a] == 0.0) {
            if (o[a] < lo[a] || o[a] >= hi[a]) { *tmin_o = INFINITY; *tmax_o = -INFINITY; return; }
        } else {
            double inv = 1.0 / d[a];
            double t0 = (lo[a] - o[a]) * inv, t1 = (hi[a] - o[a]) * inv;
            if (t0 > t1) { double t = t0; t0 = t1; t1 = t; }
            if (t0 > tmin) tmin = t0;
            if (t1 < tmax) tmax = t1;
            if (tmin > tmax) { *tmin_o = INFINITY; *tmax_o = -INFINITY; return; }
        }
    }
    *tmin_o = tmin; *tmax_o = tmax;
}

typedef struct {
    /* model, one field */
    int64_t n_bricks;
    const int32_t *blo, *blev, *bdims;
    const int64_t* boff;
    const float* vals;
    /* regions */
    int64_t n_regions;
    const double *reg_lo, *reg_hi, *reg_finest;
    const int64_t* roff;
    const int32_t* rids;
    /* cell-location split tree (optional) */
    int64_t n_tree;
    const int32_t *tx_axis, *tx_l, *tx_r, *tx_bs, *tx_bc;
    const double *tx_blo, *tx_bhi, *tx_mh;
} xo_scene_t;

static int next_hit(const xo_bvh_t* bv, const xo_scene_t* s, const double o[3], const double d[3], double t_start, double t_max,
                    double* out_in, double* out_out) {
    /* _bvh_next_hit, R/accel.py:285-352 */
    int best_r = -1;
    double best_in = INFINITY, best_out = INFINITY;
    if (bv->n_prims == 0) { *out_in = best_in; *out_out = best_out; return -1; }
    int32_t stack[256];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        int node = stack[--top];
        double n_in, n_out;
        slab(&bv->nlo[3 * node], &bv->nhi[3 * node], o, d, &n_in, &n_out);
        double lo_t = n_in > t_start ? n_in : t_start;
        double hi_t = n_out < t_max ? n_out : t_max;
        if (lo_t >= hi_t || lo_t > best_in) continue;
        if (bv->left[node] < 0) {
            int64_t st = bv->start[node];
            for (int t = 0; t < bv->count[node]; t++) {
                int r = bv->prims[st + t];
                double r_in, r_out;
                slab(&s->reg_lo[3 * r], &s->reg_hi[3 * r], o, d, &r_in, &r_out);
                double c_in = r_in > t_start ? r_in : t_start;
                double c_out = r_out < t_max ? r_out : t_max;
                if (c_in < c_out && (c_in < best_in || (c_in == best_in && r < best_r))) { best_r = r; best_in = c_in; best_out = c_out; }
            }
        } else {
            int l = bv->left[node], r = bv->right[node];
            double l_in, l_out, r_in, r_out;
            slab(&bv->nlo[3 * l], &bv->nhi[3 * l], o, d, &l_in, &l_out);
            slab(&bv->nlo[3 * r], &bv->nhi[3 * r], o, d, &r_in, &r_out);
            if (l_in <= r_in) { stack[top++] = r; stack[top++] = l; }
            else { stack[top++] = l; stack[top++] = r; }
        }
    }
    *out_in = best_in; *out_out = best_out;
    return best_r;
}

static int point_query(const xo_bvh_t* bv, const xo_scene_t* s, double px, double py, double pz) {
    /* _bvh_point_query, R/accel.py:355-388 */
    if (bv->n_prims == 0) return -1;
    int32_t stack[256];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        int node = stack[--top];
        const double *lo = &bv->nlo[3 * node], *hi = &bv->nhi[3 * node];
        if (px < lo[0] || px >= hi[0] || py < lo[1] || py >= hi[1] || pz < lo[2] || pz >= hi[2]) continue;
        if (bv->left[node] < 0) {
            int64_t st = bv->start[node];
            for (int t = 0; t < bv->count[node]; t++) {
                int r = bv->prims[st + t];
                const double *a = &s->reg_lo[3 * r], *b = &s->reg_hi[3 * r];
                if (px >= a[0] && px < b[0] && py >= a[1] && py < b[1] && pz >= a[2] && pz < b[2]) return r;
            }
        } else {
            stack[top++] = bv->right[node];
            stack[top++] = bv->left[node];
        }
    }
    return -1;
}

XO_API int xo_next_hit(const xo_bvh_t* bv, const xo_scene_t* s, const double* o, const double* d, double t_start, double t_max, double* tio) {
    return next_hit(bv, s, o, d, t_start, t_max, &tio[0], &tio[1]);
}

XO_API int xo_point_query(const xo_bvh_t* bv, const xo_scene_t* s, const double* p) { return point_query(bv, s, p[0], p[1], p[2]); }

/* ======================================================================== */
/* reconstruction  (R/sampling.py:57-224)                                   */

#define EPS_WEIGHT 1e-12

static inline void accumulate_bricks(const xo_scene_t* s, const int32_t* ids, int64_t nids, double px, double py, double pz,
                                     double* num_o, double* den_o) {
    /* _accumulate_bricks + _hat_terms, R/sampling.py:57-103 */
    double num = 0.0, den = 0.0;
    for (int64_t t = 0; t < nids; t++) {
        int64_t b = ids[t];
        int64_t lev = s->blev[b];
        double w = ldexp(1.0, (int)lev);
        int64_t iw = (int64_t)1 << lev;
        int64_t nx = s->bdims[3 * b], ny = s->bdims[3 * b + 1], nz = s->bdims[3 * b + 2];
        int64_t lx = s->blo[3 * b], ly = s->blo[3 * b + 1], lz = s->blo[3 * b + 2];
        int64_t x0 = (int64_t)floor((px - (double)lx) / w - 0.5);
        int64_t y0 = (int64_t)floor((py - (double)ly) / w - 0.5);
        int64_t z0 = (int64_t)floor((pz - (double)lz) / w - 0.5);
        int64_t base = s->boff[b];
        int64_t zs = z0 > 0 ? z0 : 0, ze = z0 + 2 < nz ? z0 + 2 : nz;
        int64_t ys = y0 > 0 ? y0 : 0, ye = y0 + 2 < ny ? y0 + 2 : ny;
        int64_t xs = x0 > 0 ? x0 : 0, xe = x0 + 2 < nx ? x0 + 2 : nx;
        for (int64_t z = zs; z < ze; z++)
            for (int64_t y = ys; y < ye; y++)
                for (int64_t x = xs; x < xe; x++) {
                    double ai = (double)(lx + x * iw), aj = (double)(ly + y * iw), ak = (double)(lz + z * iw);
                    double hx = 1.0 - fabs((ai + 0.5 * w) - px) / w;
                    double hy = 1.0 - fabs((aj + 0.5 * w) - py) / w;
                    double hz = 1.0 - fabs((ak + 0.5 * w) - pz) / w;
                    if (hx > 0.0 && hy > 0.0 && hz > 0.0) {
                        double h = hx * hy * hz;
                        num += h * (double)s->vals[base + x + nx * (y + ny * z)];
                        den += h;
                    }
                }
    }
    *num_o = num; *den_o = den;
}

static inline void gradient_bricks(const xo_scene_t* s, const int32_t* ids, int64_t nids, double px, double py, double pz, double out[8]) {
    /* _gradient_bricks, R/sampling.py:123-181 */
    double num = 0.0, den = 0.0, dnx = 0.0, dny = 0.0, dnz = 0.0, ddx = 0.0, ddy = 0.0, ddz = 0.0, v0 = 0.0;
    int have_ref = 0;
    for (int64_t t = 0; t < nids; t++) {
        int64_t b = ids[t];
        int64_t lev = s->blev[b];
        double w = ldexp(1.0, (int)lev);
        int64_t iw = (int64_t)1 << lev;
        int64_t nx = s->bdims[3 * b], ny = s->bdims[3 * b + 1], nz = s->bdims[3 * b + 2];
        int64_t lx = s->blo[3 * b], ly = s->blo[3 * b + 1], lz = s->blo[3 * b + 2];
        int64_t x0 = (int64_t)floor((px - (double)lx) / w - 0.5);
        int64_t y0 = (int64_t)floor((py - (double)ly) / w - 0.5);
        int64_t z0 = (int64_t)floor((pz - (double)lz) / w - 0.5);
        int64_t base = s->boff[b];
        int64_t zs = z0 > 0 ? z0 : 0, ze = z0 + 2 < nz ? z0 + 2 : nz;
        int64_t ys = y0 > 0 ? y0 : 0, ye = y0 + 2 < ny ? y0 + 2 : ny;
        int64_t xs = x0 > 0 ? x0 : 0, xe = x0 + 2 < nx ? x0 + 2 : nx;
        for (int64_t z = zs; z < ze; z++)
            for (int64_t y = ys; y < ye; y++)
                for (int64_t x = xs; x < xe; x++) {
                    double ai = (double)(lx + x * iw), aj = (double)(ly + y * iw), ak = (double)(lz + z * iw);
                    double hx = 1.0 - fabs((ai + 0.5 * w) - px) / w;
                    double hy = 1.0 - fabs((aj + 0.5 * w) - py) / w;
                    double hz = 1.0 - fabs((ak + 0.5 * w) - pz) / w;
                    if (hx > 0.0 && hy > 0.0 && hz > 0.0) {
                        double sx = (ai + 0.5 * w) - px > 0.0 ? 1.0 : -1.0;
                        double sy = (aj + 0.5 * w) - py > 0.0 ? 1.0 : -1.0;
                        double sz = (ak + 0.5 * w) - pz > 0.0 ? 1.0 : -1.0;
                        double gx = sx / w * hy * hz, gy = sy / w * hx * hz, gz = sz / w * hx * hy;
                        double h = hx * hy * hz;
                        double v = (double)s->vals[base + x + nx * (y + ny * z)];
                        if (!have_ref) { v0 = v; have_ref = 1; }
                        double u = v - v0;
                        num += h * u; den += h;
                        dnx += gx * u; dny += gy * u; dnz += gz * u;
                        ddx += gx; ddy += gy; ddz += gz;
                    }
                }
    }
    out[0] = num; out[1] = den; out[2] = dnx; out[3] = dny; out[4] = dnz; out[5] = ddx; out[6] = ddy; out[7] = ddz;
}

static int collect_bricks(const xo_scene_t* s, double px, double py, double pz, int32_t* out, int cap) {
    /* _collect_bricks, R/sampling.py:184-224 */
    int n = 0;
    int32_t stack[256];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
        int nd = stack[--top];
        double e = s->tx_mh[nd];
        const double *lo = &s->tx_blo[3 * nd], *hi = &s->tx_bhi[3 * nd];
        if (px <= lo[0] - e || px >= hi[0] + e || py <= lo[1] - e || py >= hi[1] + e || pz <= lo[2] - e || pz >= hi[2] + e) continue;
        if (s->tx_axis[nd] < 0) {
            for (int b = s->tx_bs[nd]; b < s->tx_bs[nd] + s->tx_bc[nd]; b++) if (n < cap) out[n++] = b;
        } else {
            stack[top++] = s->tx_r[nd];
            stack[top++] = s->tx_l[nd];
        }
    }
    for (int a = 1; a < n; a++) {
        int32_t key = out[a];
        int c = a - 1;
        while (c >= 0 && out[c] > key) { out[c + 1] = out[c]; c--; }
        out[c + 1] = key;
    }
    return n;
}

/* point API: region sample, oracle scan, gradients */
XO_API void xo_sample_region(const xo_scene_t* s, int64_t rid, const double* p, double* out) {
    double num, den;
    accumulate_bricks(s, s->rids + s->roff[rid], s->roff[rid + 1] - s->roff[rid], p[0], p[1], p[2], &num, &den);
    out[0] = num; out[1] = den;
}

XO_API void xo_sample_brick_list(const xo_scene_t* s, const int32_t* ids, int64_t nids, const double* p, double* out) {
    accumulate_bricks(s, ids, nids, p[0], p[1], p[2], &out[0], &out[1]);
}

XO_API void xo_sample_cells(int64_t n, const int32_t* ci, const int32_t* cj, const int32_t* ck, const int32_t* clev, const float* cvals,
                            const double* p, double* out) {
    /* _accumulate_cells, R/sampling.py:106-120 */
    double num = 0.0, den = 0.0;
    for (int64_t t = 0; t < n; t++) {
        double w = ldexp(1.0, clev[t]);
        double hx = 1.0 - fabs(((double)ci[t] + 0.5 * w) - p[0]) / w;
        double hy = 1.0 - fabs(((double)cj[t] + 0.5 * w) - p[1]) / w;
        double hz = 1.0 - fabs(((double)ck[t] + 0.5 * w) - p[2]) / w;
        if (hx > 0.0 && hy > 0.0 && hz > 0.0) {
            double h = hx * hy * hz;
            num += h * (double)cvals[t];
            den += h;
        }
    }
    out[0] = num; out[1] = den;
}

XO_API void xo_gradient_region(const xo_scene_t* s, int64_t rid, const double* p, double* out) {
    gradient_bricks(s, s->rids + s->roff[rid], s->roff[rid + 1] - s->roff[rid], p[0], p[1], p[2], out);
}

XO_API int xo_collect_bricks(const xo_scene_t* s, const double* p, int32_t* out, int cap) { return collect_bricks(s, p[0], p[1], p[2], out, cap); }

/* ======================================================================== */
/* renderer  (R/render.py:226-578)                                          */

typedef struct {
    int32_t width, height;
    double pos[3], right[3], up[3], fwd[3];
    double tan_half, aspect;
} xo_camera_t;

typedef struct {
    double spc, rate, early;
    uint64_t seed;
    int32_t grad_mode, n_planes;
    double planes[6][4];
    int32_t iso_on, use_tree;
    double iso_value, iso_rgb[3];
    double tf_lo, tf_hi;
    const double* tf_rgba;
} xo_march_t;

static inline double rho_hash(uint64_t pixel, uint64_t seed) {
    /* _rho_hash, R/render.py:226-233 */
    uint64_t z = pixel ^ seed;
    z = z + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

XO_API double xo_rho(uint64_t pixel, uint64_t seed) { return rho_hash(pixel, seed); }

static inline double restart_t(double t_out) { double e = 1e-7 * t_out; return t_out + (e > 1e-7 ? e : 1e-7); }

static int clip_ray(const xo_march_t* m, const double o[3], const double d[3], double* tmin, double* tmax) {
    /* _clip_ray, R/render.py:263-281 */
    for (int i = 0; i < m->n_planes; i++) {
        const double* pl = m->planes[i];
        double nd = pl[0] * d[0] + pl[1] * d[1] + pl[2] * d[2];
        double no = pl[0] * o[0] + pl[1] * o[1] + pl[2] * o[2];
        if (nd > 0.0) { double t = (pl[3] - no) / nd; if (t < *tmax) *tmax = t; }
        else if (nd < 0.0) { double t = (pl[3] - no) / nd; if (t > *tmin) *tmin = t; }
        else if (no > pl[3]) { *tmin = 1.0; *tmax = 0.0; return 0; }
    }
    return 1;
}

static inline double shade_factor(double gx, double gy, double gz, const double d[3]) {
    double n = sqrt(gx * gx + gy * gy + gz * gz);
    if (n == 0.0) return 0.2;
    return 0.2 + 0.8 * fabs(gx * d[0] + gy * d[1] + gz * d[2]) / n;
}

static void sample_gradient(const xo_scene_t* s, const xo_bvh_t* ab, int grad_mode, double px, double py, double pz, int rid,
                            const int32_t* ids, int64_t nids, double val, double g[3]) {
    /* _sample_gradient, R/render.py:292-377 */
    if (grad_mode == 1) {
        double a[8];
        gradient_bricks(s, ids, nids, px, py, pz, a);
        if (a[1] <= EPS_WEIGHT) { g[0] = g[1] = g[2] = 0.0; return; }
        double d2 = a[1] * a[1];
        g[0] = (a[2] * a[1] - a[0] * a[5]) / d2;
        g[1] = (a[3] * a[1] - a[0] * a[6]) / d2;
        g[2] = (a[4] * a[1] - a[0] * a[7]) / d2;
        return;
    }
    double h = 0.5 * s->reg_finest[rid];
    double p[3] = {px, py, pz};
    g[0] = g[1] = g[2] = 0.0;
    for (int a = 0; a < 3; a++) {
        double qp[3] = {px, py, pz}, qm[3] = {px, py, pz};
        qp[a] = p[a] + h;
        qm[a] = p[a] - h;
        if (grad_mode == 3) {
            const double *lo = &s->reg_lo[3 * rid], *hi = &s->reg_hi[3 * rid];
            for (int c = 0; c < 3; c++) {
                qp[c] = fmin(fmax(qp[c], lo[c]), hi[c]);
                qm[c] = fmin(fmax(qm[c], lo[c]), hi[c]);
            }
            double np_, dp, nm, dm;
            accumulate_bricks(s, ids, nids, qp[0], qp[1], qp[2], &np_, &dp);
            accumulate_bricks(s, ids, nids, qm[0], qm[1], qm[2], &nm, &dm);
            if (dp > EPS_WEIGHT && dm > EPS_WEIGHT) {
                double span = qp[a] - qm[a];
                if (span > 0.0) g[a] = (np_ / dp - nm / dm) / span;
            }
        } else {
            double fp = 0.0, fm = 0.0;
            int okp = 0, okm = 0;
            int rp = point_query(ab, s, qp[0], qp[1], qp[2]);
            if (rp >= 0) {
                double n_, d_;
                accumulate_bricks(s, s->rids + s->roff[rp], s->roff[rp + 1] - s->roff[rp], qp[0], qp[1], qp[2], &n_, &d_);
                if (d_ > EPS_WEIGHT) { fp = n_ / d_; okp = 1; }
            }
            int rm = point_query(ab, s, qm[0], qm[1], qm[2]);
            if (rm >= 0) {
                double n_, d_;
                accumulate_bricks(s, s->rids + s->roff[rm], s->roff[rm + 1] - s->roff[rm], qm[0], qm[1], qm[2], &n_, &d_);
                if (d_ > EPS_WEIGHT) { fm = n_ / d_; okm = 1; }
            }
            double gg;
            if (okp && okm) gg = (fp - fm) / (2.0 * h);
            else if (okp) gg = (fp - val) / h;
            else if (okm) gg = (val - fm) / h;
            else gg = 0.0;
            g[a] = gg;
        }
    }
}

static void volume_ray(const xo_scene_t* s, const xo_bvh_t* vb, const xo_bvh_t* ab, const xo_march_t* m, const double o[3], const double d[3],
                       double tmin, double tmax, double rho, double acc[4], int64_t* n_reg, int64_t* n_smp) {
    /* _volume_ray, R/render.py:380-453 */
    double ar = 0.0, ag = 0.0, abl = 0.0, aa = 0.0;
    int64_t nr = 0, ns = 0;
    double t = tmin;
    int32_t tbuf[1024];
    while (aa < m->early) {
        double t_in, t_out;
        int rid = next_hit(vb, s, o, d, t, tmax, &t_in, &t_out);
        if (rid < 0) break;
        nr++;
        double fw = s->reg_finest[rid];
        double dt = fw / (m->spc * m->rate);
        double s1 = fw / m->spc;
        const int32_t* ids = s->rids + s->roff[rid];
        int64_t nids = s->roff[rid + 1] - s->roff[rid];
        double prev = t_in;
        double k = floor(t_in / dt - rho) + 1.0;
        int done = 0;
        while (!done) {
            double tk = dt * (k + rho);
            k += 1.0;
            if (tk >= t_out) { tk = t_out; done = 1; }
            else if (tk <= prev) continue;
            double sl = tk - prev;
            double mid = 0.5 * (prev + tk);
            prev = tk;
            ns++;
            double px = o[0] + mid * d[0], py = o[1] + mid * d[1], pz = o[2] + mid * d[2];
            double num, den;
            if (m->use_tree) {
                int nb = collect_bricks(s, px, py, pz, tbuf, 1024);
                accumulate_bricks(s, tbuf, nb, px, py, pz, &num, &den);
            } else {
                accumulate_bricks(s, ids, nids, px, py, pz, &num, &den);
            }
            if (den > EPS_WEIGHT) {
                double v = num / den;
                double c[4];
                tf_eval(m->tf_lo, m->tf_hi, m->tf_rgba, v, c);
                if (c[3] > 0.0) {
                    double alpha = 1.0 - pow(1.0 - c[3], sl / s1);
                    if (m->grad_mode != 0) {
                        double g[3];
                        sample_gradient(s, ab, m->grad_mode, px, py, pz, rid, ids, nids, v, g);
                        double f = shade_factor(g[0], g[1], g[2], d);
                        c[0] *= f; c[1] *= f; c[2] *= f;
                    }
                    double w = alpha * (1.0 - aa);
                    ar += w * c[0]; ag += w * c[1]; abl += w * c[2]; aa += w;
                    if (aa >= m->early) break;
                }
            }
        }
        t = restart_t(t_out);
        if (t >= tmax) break;
    }
    acc[0] = ar; acc[1] = ag; acc[2] = abl; acc[3] = aa;
    *n_reg = nr; *n_smp = ns;
}

static int iso_ray(const xo_scene_t* s, const xo_bvh_t* ib, const xo_march_t* m, const double o[3], const double d[3], double tmin, double tmax,
                   double rho, double* t_hit_o, double g[3]) {
    /* _iso_ray, R/render.py:456-518 */
    double t = tmin, iso = m->iso_value;
    g[0] = g[1] = g[2] = 0.0;
    for (;;) {
        double t_in, t_out;
        int rid = next_hit(ib, s, o, d, t, tmax, &t_in, &t_out);
        if (rid < 0) return 0;
        double fw = s->reg_finest[rid];
        double dt = fw / (m->spc * m->rate);
        const int32_t* ids = s->rids + s->roff[rid];
        int64_t nids = s->roff[rid + 1] - s->roff[rid];
        double prev_t = t_in, num, den;
        accumulate_bricks(s, ids, nids, o[0] + t_in * d[0], o[1] + t_in * d[1], o[2] + t_in * d[2], &num, &den);
        int prev_ok = den > EPS_WEIGHT;
        double prev_f = prev_ok ? num / den - iso : 0.0;
        double k = floor(t_in / dt - rho) + 1.0;
        int done = 0;
        while (!done) {
            double tk = dt * (k + rho);
            k += 1.0;
            if (tk >= t_out) { tk = t_out; done = 1; }
            else if (tk <= prev_t) continue;
            accumulate_bricks(s, ids, nids, o[0] + tk * d[0], o[1] + tk * d[1], o[2] + tk * d[2], &num, &den);
            int ok = den > EPS_WEIGHT;
            double f = ok ? num / den - iso : 0.0;
            if (prev_ok && ok && ((prev_f <= 0.0 && f >= 0.0) || (prev_f >= 0.0 && f <= 0.0)) && !(prev_f == 0.0 && f == 0.0)) {
                double lo_t = prev_t, hi_t = tk, flo = prev_f;
                for (int it = 0; it < 16; it++) {
                    double mid = 0.5 * (lo_t + hi_t);
                    accumulate_bricks(s, ids, nids, o[0] + mid * d[0], o[1] + mid * d[1], o[2] + mid * d[2], &num, &den);
                    double fm = den > EPS_WEIGHT ? num / den - iso : 0.0;
                    if ((flo <= 0.0 && fm <= 0.0) || (flo >= 0.0 && fm >= 0.0)) { lo_t = mid; flo = fm; }
                    else hi_t = mid;
                }
                double th = 0.5 * (lo_t + hi_t);
                *t_hit_o = th;
                double a[8];
                gradient_bricks(s, ids, nids, o[0] + th * d[0], o[1] + th * d[1], o[2] + th * d[2], a);
                if (a[1] > EPS_WEIGHT) {
                    double d2 = a[1] * a[1];
                    g[0] = (a[2] * a[1] - a[0] * a[5]) / d2;
                    g[1] = (a[3] * a[1] - a[0] * a[6]) / d2;
                    g[2] = (a[4] * a[1] - a[0] * a[7]) / d2;
                }
                return 1;
            }
            prev_t = tk; prev_f = f; prev_ok = ok;
        }
        t = restart_t(t_out);
        if (t >= tmax) return 0;
    }
}

static void render_pixel(const xo_scene_t* s, const xo_bvh_t* vb, const xo_bvh_t* ib, const xo_bvh_t* ab, const xo_camera_t* cam,
                         const xo_march_t* m, int64_t pix, double out[4], int64_t* nreg, int64_t* nsmp) {
    /* per-pixel body of _render_kernel, R/render.py:525-578 */
    int64_t W = cam->width, H = cam->height;
    int64_t x = pix % W, y = pix / W;
    double sx = (2.0 * ((double)x + 0.5) / (double)W - 1.0) * cam->tan_half * cam->aspect;
    double sy = (1.0 - 2.0 * ((double)y + 0.5) / (double)H) * cam->tan_half;
    double d[3];
    for (int a = 0; a < 3; a++) d[a] = cam->fwd[a] + sx * cam->right[a] + sy * cam->up[a];
    double inv = 1.0 / sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    d[0] *= inv; d[1] *= inv; d[2] *= inv;
    const double* o = cam->pos;
    double rho = rho_hash((uint64_t)pix, m->seed);
    double tmin = 0.0, tmax = 1.0e30;
    clip_ray(m, o, d, &tmin, &tmax);
    if (tmin >= tmax) { out[0] = out[1] = out[2] = out[3] = 0.0; *nreg = 0; *nsmp = 0; return; }
    double t_end = tmax, g[3] = {0, 0, 0}, t_hit = 0.0;
    int hit = 0;
    if (m->iso_on) {
        hit = iso_ray(s, ib, m, o, d, tmin, tmax, rho, &t_hit, g);
        if (hit) t_end = t_hit;
    }
    double acc[4];
    volume_ray(s, vb, ab, m, o, d, tmin, t_end, rho, acc, nreg, nsmp);
    if (hit) {
        double f = shade_factor(g[0], g[1], g[2], d);
        double w = 1.0 - acc[3];
        acc[0] += w * m->iso_rgb[0] * f;
        acc[1] += w * m->iso_rgb[1] * f;
        acc[2] += w * m->iso_rgb[2] * f;
        acc[3] = 1.0;
    }
    for (int c = 0; c < 4; c++) out[c] = acc[c];
}

static inline uint8_t quant(double v) {
    double c = v < 0.0 ? 0.0 : v;
    c = c > 1.0 ? 1.0 : c;
    return (uint8_t)(c * 255.0 + 0.5);
}

XO_API int xo_render(const xo_scene_t* s, const xo_bvh_t* vb, const xo_bvh_t* ib, const xo_bvh_t* ab, const xo_camera_t* cam,
                     const xo_march_t* m, int64_t pix_begin, int64_t pix_end, double* out_f, uint8_t* out_u8,
                     int64_t* px_regions, int64_t* px_samples, int n_threads) {
    /* out_* are indexed by (pix - pix_begin) */
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int64_t pix = pix_begin; pix < pix_end; pix++) {
        double o4[4];
        int64_t nr, ns;
        render_pixel(s, vb, ib, ab, cam, m, pix, o4, &nr, &ns);
        int64_t q = pix - pix_begin;
        if (out_f) for (int c = 0; c < 4; c++) out_f[4 * q + c] = o4[c];
        if (out_u8) for (int c = 0; c < 4; c++) out_u8[4 * q + c] = quant(o4[c]);
        if (px_regions) px_regions[q] = nr;
        if (px_samples) px_samples[q] = ns;
    }
    return 0;
}

XO_API void xo_integrate_ray(const xo_scene_t* s, const xo_bvh_t* vb, const xo_bvh_t* ab, const xo_march_t* m, const double* o, const double* d,
                             double tmin, double tmax, double rho, double* out, int64_t* counts) {
    /* integrate_ray body, R/render.py:613-632 (direction already normalised by the caller) */
    clip_ray(m, o, d, &tmin, &tmax);
    if (tmin >= tmax) { out[0] = out[1] = out[2] = out[3] = 0.0; counts[0] = counts[1] = 0; return; }
    volume_ray(s, vb, ab, m, o, d, tmin, tmax, rho, out, &counts[0], &counts[1]);
}

XO_API int xo_iso_intersect(const xo_scene_t* s, const xo_bvh_t* ib, const xo_march_t* m, const double* o, const double* d, double tmin,
                            double tmax, double rho, double* out) {
    double g[3], th = 0.0;
    int hit = iso_ray(s, ib, m, o, d, tmin, tmax, rho, &th, g);
    out[0] = th; out[1] = g[0]; out[2] = g[1]; out[3] = g[2];
    return hit;
}

XO_API int xo_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
