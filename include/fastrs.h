/*
 * fastrs.h — C ABI of the B200 (sm_100a) local-thickness sphericity/roundness library
 * (libfastrs.so).  Method: arXiv 2504.05808 ("fast_rs"), §4.
 *
 * The problem statement follows the paper: given a mask of many labelled objects, compute
 * sphericity and roundness for all objects at once from ONE local-thickness pass
 * (§1, §4, §5.3).  Four stages, all in hand-written
 * CUDA kernels:
 *   1. exact label-aware squared EDT  D(p)      (substrate of LT)
 *   2. local thickness LT^2(p) = max{D(q): |p-q|^2 < D(q)}  (radius, c3)
 *   3. shell (4/6-connected contour) + per-label segmented reductions:
 *      V, mean LT (a_s / a_e), max LT (R),
 *      mean shell LT (r_bar)
 *   4. closed forms: 3D Eqs. 1,6,7,8, 2D Eqs. 2,9,10,11
 *      (PAPER.md:45-48,129-137), roundness R = r_bar / R_max.
 * Readings of silent/garbled passages (eccentricity form, label-aware sites, border
 * convention, ...) are listed in DESIGN.md "Readings" and follow SURVEY.md §8(c).
 *
 * Conventions (all entry points)
 *  - labels: int32, C order.  ndim = 3: dims = {Z, Y, X}; ndim = 2: dims = {Y, X}.
 *    batch >= 1 independent images/volumes are stacked outermost: [batch][Z][Y][X].
 *    0 = background; objects are labels 1..max_label, independent per batch item.
 *  - Every element with a different label (other objects included) is a site of an
 *    object's distance transform; with FASTRS_BORDER_BACKGROUND the virtual layer just
 *    outside the grid is a site too (and counts as a background neighbour for the shell).
 *  - All data pointers are DEVICE pointers owned by the caller (except the _host entry
 *    point and the pure math functions).  Work is enqueued on `stream` (a cudaStream_t;
 *    NULL = legacy default stream).  By default each call synchronises the stream once,
 *    at its end, to read a 4-byte status word; FASTRS_ASYNC skips that synchronisation
 *    (the status then stays in the workspace: read it with fastrs_read_diagnostics).
 *  - `ws` is caller-owned device scratch of at least fastrs_workspace_bytes() bytes,
 *    256-byte aligned.  The library allocates nothing per call; it keeps one per-device
 *    cache (lattice containment table, ~0.6 MB) until fastrs_release().
 *  - Limits: every dim in [1, 16384]; X <= 16384; squared distances < 2^30.
 *  - Return value: a fastrs_status.  On a non-OK return fastrs_last_error() gives a
 *    thread-local message.  Outputs are unspecified after a non-OK return.
 *  - Per-label outputs have batch*max_label entries, index b*max_label + (label-1).
 *    Labels absent from an item (V = 0) get NaN metrics and zero counts.
 */
#ifndef FASTRS_H
#define FASTRS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FASTRS_API __attribute__((visibility("default")))
#else
#define FASTRS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FASTRS_OK = 0,
  FASTRS_EINVAL = 1,    /* bad argument: ndim not 2/3, dim < 1 or > 16384, batch < 1, null
                           pointer, label < 0 or > max_label (SPEC.md:48 invalid-argument) */
  FASTRS_ENOSITE = 2,   /* some object element has no site at all (an object fills every
                           line it lies on and the border is not background) */
  FASTRS_ENOMEM = 3,    /* ws_bytes smaller than fastrs_workspace_bytes() */
  FASTRS_ECUDA = 4,     /* a CUDA runtime error (message in fastrs_last_error) */
  FASTRS_ENCCL = 5,     /* an NCCL call of the multi-GPU slab path failed (or NCCL is missing) */
  FASTRS_EINTERNAL = 6  /* a device-side invariant failed (e.g. LT^2 < D) */
} fastrs_status;

enum {
  FASTRS_BORDER_BACKGROUND = 1u, /* the grid border is background   */
  FASTRS_DETERMINISTIC = 2u,     /* accepted for compatibility: sums are ALWAYS exact
                                    fixed-point integers, bit-identical across runs     */
  FASTRS_ASYNC = 4u,             /* do not synchronise the stream at the end of the call  */
  FASTRS_HOST_IO = 8u,           /* size the workspace for fastrs_sphericity_roundness_host */
  FASTRS_FORCE_FALLBACK = 16u,   /* run K5 with the atomic sparse-table kernel on every tile
                                    (a GPU-internal cross-check of the default dilation)    */
  FASTRS_EDGE_SKIP_ZLO = 32u,    /* fastrs_touches_edge on a z-slab (3D): its first slice is  */
  FASTRS_EDGE_SKIP_ZHI = 64u,    /* not a grid face / its last slice is not (slab path)      */
  FASTRS_SLAB_TRANSPOSE = 128u,  /* fastrs_sphericity_roundness_slab: z pass by the all-to-all
                                    z-slab -> y-slab transpose (N1) instead of the h halo (N8) */
  FASTRS_SLAB_DENSE_HALO = 512u, /* fastrs_sphericity_roundness_slab: exchange H dense slices of D
                                    for the dilation instead of the kept-centre halo (N4)        */
  FASTRS_NO_LIST_STAGING = 1024u,/* test hook: a K5 candidate list that overflows the shared list is
                                    regathered (a second pass) instead of staged in the pool      */
  FASTRS_EXACT_PRUNE = 4096u,    /* K4 tests every offset class with |s|^2 <= 12 (the exact lattice
                                    maximal-ball set for that stencil).  Default:
                                    the 26-neighbourhood and the five stage-2 classes that drop
                                    centres on C4 -- a superset of kept balls, LT^2 unchanged      */
  FASTRS_NO_COVER_CUT = 2048u,   /* test hook: K5a keeps every ball that reaches a tile group even
                                    when the largest one contains all of its foreground (the cut
                                    is exact; this exercises the long-list paths it avoids)       */
  FASTRS_APPROX_LT = 256u        /* approximate local thickness (SPEC.md:153
                                    local_thickness_fast): each 2048-element tile stops its exact
                                    cover once at most 4 % of its foreground is uncovered, and those
                                    cells take LT^2 = D (their own ball).  Guarantees D <= LT^2_fast
                                    <= LT^2, LT^2_fast <= the object's max D, and >= 96 % of every
                                    tile's foreground exact (so >= 95 % within 5 %). */
};

/* u32 words per tile record of fastrs_slab_pack_tiles / fastrs_slab_unpack_tiles. */
#define FASTRS_TILE_RECORD_WORDS 20

/* Optional per-label statistics (device pointers, each nullable, batch*max_label long). */
typedef struct {
  int64_t* volume;        /* V (3D) or A (2D): element count           */
  int64_t* n_shell;       /* number of shell elements (D == 1 <=> face neighbour ≠)  */
  uint32_t* max_lt2;      /* max LT^2 = max D (exact integer)                         */
  double* mean_lt;        /* a_s / a_e: mean of sqrt(LT^2) over the object            */
  double* max_lt;         /* R = sqrt(max_lt2)                                        */
  double* shell_mean_lt;  /* r_bar: mean of sqrt(LT^2) over the shell                 */
  double* axis_a;         /* model semi-axis a (= mean_lt)                            */
  double* axis_cb;        /* c_s = 3V/(4 pi a^2) (Eq. 8) or b_e = A/(pi a) (Eq. 10)   */
} fastrs_object_stats;

/* Counters left in the workspace by the last call that used it (diagnostics / bench). */
typedef struct {
  uint32_t status_bits;   /* bit0 bad label, bit1 no site, bit2 LT2<D, bit3 shell        */
  uint32_t dmax;          /* max squared distance over the grid                          */
  uint64_t n_fg;          /* foreground elements                                         */
  uint64_t n_kept;        /* maximal-ball centres kept by the lattice pruning (K4)       */
  uint64_t n_intervals;   /* (ball, row) chords the dilation (K5) evaluated exactly       */
  int32_t sum_scale_log2; /* fixed-point scale of the LT sums (2^s)                      */
  uint32_t n_fallback;   /* tile groups handed to the atomic fallback dilation         */
  uint32_t n_rounds_extra; /* K5: candidate-list rounds beyond the first, summed over groups */
  uint32_t n_regathers;  /* K5: list overflows that needed a second gather pass         */
  uint32_t max_group_list; /* K5: longest per-group candidate list                      */
  uint64_t sum_group_list; /* K5: candidates summed over tile groups                    */
  uint64_t n_painted;      /* K5: balls painted row-parallel after the screens (S&R call) */
  uint64_t n_covering;     /* K5: painted balls that covered at least one cell (S&R call) */
  uint32_t n_staged;       /* K5: list overflows staged in the candidate pool (one pass)   */
  uint32_t n_deferred;     /* K5: tile groups a full candidate pool deferred to a later wave */
  uint32_t n_col_slow;     /* last column pass (K3 in 3D): elements whose scan left the staged
                              window, scanned by the batched-read list kernel              */
  uint32_t reserved;
} fastrs_diagnostics;

/* Bytes of device workspace needed by every entry point below for this geometry.
 * max_label may be 0 for edt/LT-only use.  flags: FASTRS_HOST_IO adds room for the
 * labels and outputs of fastrs_sphericity_roundness_host.  Returns FASTRS_OK/EINVAL. */
FASTRS_API int fastrs_workspace_bytes(const int64_t* dims, int ndim, int64_t batch, int32_t max_label,
                           uint32_t flags, size_t* bytes);

/* Stage 1 only: exact squared label-aware EDT.  d2_out: uint32 [batch][Z][Y][X] (device),
 * 0 on background, D >= 1 on objects. */
FASTRS_API int fastrs_edt_sq(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                  uint32_t flags, uint32_t* d2_out, void* ws, size_t ws_bytes, void* stream);

/* Stages 1-2: exact local thickness.  lt2_out: uint32 LT^2 (nullable); lt_out: float32
 * LT radius = (float)sqrt((double)LT^2) (nullable); at least one non-null; both 0 on
 * background. */
FASTRS_API int fastrs_local_thickness(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                           uint32_t flags, uint32_t* lt2_out, float* lt_out, void* ws,
                           size_t ws_bytes, void* stream);

/* Stages 1-4: per-object sphericity and roundness for every label 1..max_label of every
 * batch item.  sphericity, roundness: float64 device arrays of batch*max_label (either may
 * be NULL); stats: optional host struct of device pointers (NULL = none).
 * (§4.1-4.2) */
FASTRS_API int fastrs_sphericity_roundness(const int32_t* labels, const int64_t* dims, int ndim,
                                int64_t batch, int32_t max_label, uint32_t flags,
                                double* sphericity, double* roundness,
                                const fastrs_object_stats* stats, void* ws, size_t ws_bytes,
                                void* stream);

/* Same as fastrs_sphericity_roundness with HOST buffers: labels_host (ideally pinned) is
 * copied to the device inside the call, results are copied back to sphericity_host /
 * roundness_host (batch*max_label float64 each, nullable) before it returns.  The
 * workspace must be sized with FASTRS_HOST_IO.  Always synchronises.  This is the
 * end-to-end ("e2e") entry point timed by bench.py. */
FASTRS_API int fastrs_sphericity_roundness_host(const int32_t* labels_host, const int64_t* dims, int ndim,
                                     int64_t batch, int32_t max_label, uint32_t flags,
                                     double* sphericity_host, double* roundness_host, void* ws,
                                     size_t ws_bytes, void* stream);

/* Copy the diagnostics counters of the last call on `ws` to the host (synchronises). */
FASTRS_API int fastrs_read_diagnostics(const void* ws, fastrs_diagnostics* out, void* stream);

/* Per-stage device time (ms) accumulated over calls while profiling is on: stages are
 * 0 edt_x, 1 edt_y, 2 edt_z, 3 prune, 4 dilate (K5b paint + fallback), 5 metrics, 6 epilogue
 * (K5 shell + reductions), 7 gather (K5a candidate gather + sort).
 * Events are recorded on the
 * call's stream.  fastrs_profile(1) enables and resets; fastrs_profile(0) disables. */
FASTRS_API void fastrs_profile(int enable);
FASTRS_API int fastrs_profile_read(double* ms_out, int64_t* calls_out, int n_stages);

/* Host-callable closed forms, the same __host__ __device__ code as the metrics kernel. */
FASTRS_API double fastrs_spheroid_area(double a, double c);         /* Eqs. 6-7, reading c1/c12 */
FASTRS_API double fastrs_ramanujan_perimeter(double a, double b);   /* Eq. 9                    */
FASTRS_API double fastrs_sphericity_3d(double V, double mean_lt);   /* Eqs. 1, 8                */
FASTRS_API double fastrs_sphericity_2d(double A, double mean_lt);   /* Eqs. 2, 10, 11           */

/* ---- multi-GPU z-slab path (north_star "a single large volume is
 * split into z-slabs") ------------------------------------------------------------------
 * One 3D volume [Z][Y][X] split into z-slabs, one per rank (batch = 1, ndim = 3).  Every
 * computation runs in the kernels; the caller performs the three exchanges between the phase
 * calls (paper_2504_05808_b200/slab.py does them with torch.distributed: NCCL on GPUs, gloo in
 * the CPU tests).  With h = ceil(sqrt(max D_xy)) and R = isqrt(max D - 1):
 *   A fastrs_slab_edt_xy   x and y passes of the own slab -> packed words + max D_xy
 *     exchange 1: allreduce(max) of D_xy; every rank fetches the h packed slices on each side
 *   B fastrs_slab_edt_z    z pass on the h-extended slab  -> D of the own slab + max D
 *     exchange 2: allreduce(max) of D; every rank fetches H >= R D-slices on each side
 *   C fastrs_slab_reduce   K4 on the H-extended slab, K5 + shell + partial per-label sums on the
 *                          own slab (u64 fixed-point sums, u32 max LT^2: exact integers)
 *     exchange 3: allreduce(sum) of the u64 partials, allreduce(max) of max LT^2
 *   D fastrs_metrics_from_partials   closed forms per label
 * Exactness: the z pass at an own element only looks |dz| <= sqrt(D_xy) <= h away; a ball that
 * reaches the own slab has its centre within R <= H slices; partial sums are integers, so the
 * result is bit-identical to fastrs_sphericity_roundness on the whole volume.
 * All pointers are device pointers; each phase synchronises once unless FASTRS_ASYNC. */

/* Workspace for the slab phases, sized by the extended slab dims {nz_ext, Y, X}. */
FASTRS_API int fastrs_slab_workspace_bytes(const int64_t* dims_ext, size_t* bytes);

/* A: labels = own slab [nz][Y][X] (dims = {nz, Y, X}); labels_below = the slice z0-1 of the
 * rank below ([Y][X]), NULL at the bottom of the volume.  packed_out: [nz][Y][X] u32 words
 * (partial squared distance + z-run-start flag); dxy_max (nullable): device u32 <- max partial
 * distance over the slab.  Validates labels (EINVAL). */
FASTRS_API int fastrs_slab_edt_xy(const int32_t* labels, const int32_t* labels_below, const int64_t* dims,
                                  int32_t max_label, uint32_t flags, uint32_t* packed_out, uint32_t* dxy_max,
                                  void* ws, size_t ws_bytes, void* stream);

/* B: packed_ext = packed words of global slices [z_ext0, z_ext0 + nz_ext) (dims_ext = {nz_ext, Y,
 * X}); the own slab is local [own_lo, own_hi).  d_out: [own_hi-own_lo][Y][X] squared distances;
 * dmax_out (nullable): device u32 <- max D over the own slab.  ENOSITE as fastrs_edt_sq. */
FASTRS_API int fastrs_slab_edt_z(const uint32_t* packed_ext, const int64_t* dims_ext, int64_t own_lo,
                                 int64_t own_hi, int64_t z_ext0, int64_t Z, uint32_t flags, uint32_t* d_out,
                                 uint32_t* dmax_out, void* ws, size_t ws_bytes, void* stream);

/* C: labels = own slab; d_ext = D of the extended slab (dims_ext), own slab local [own_lo,
 * own_hi), own_lo a multiple of 8 and own_hi a multiple of 8 or nz_ext; Z = global depth;
 * dmax_global = max D over the whole volume.  Writes the own slab's partial per-label sums to
 * vol, n_shell, sum_lt, sum_shell_lt (u64, fixed point 2^s with s from (Z*Y*X, dmax_global))
 * and max_lt2 (u32), each max_label long (zeroed by the call). */
FASTRS_API int fastrs_slab_reduce(const int32_t* labels, const uint32_t* d_ext, const int64_t* dims_ext,
                                  int64_t own_lo, int64_t own_hi, int64_t Z, uint32_t dmax_global,
                                  int32_t max_label, uint32_t flags, uint64_t* vol, uint64_t* n_shell,
                                  uint64_t* sum_lt, uint64_t* sum_shell_lt, uint32_t* max_lt2, void* ws,
                                  size_t ws_bytes, void* stream);

/* C, split for the kept-centre halo (N4: instead of the H slices of D, neighbours exchange the
 * K4 outputs of the tile layers within H slices of each other's slab):
 *   fastrs_slab_prune   K4 on the own tile layers only (d_ext must hold D of the own slab and the
 *                       3 slices on each side that K4's |s|^2 <= 12 stencil reads; the other
 *                       layers' tile data are cleared)
 *   fastrs_slab_pack_tiles / fastrs_slab_unpack_tiles   the K4 outputs of tile layers
 *                       [tz_a, tz_b) of the extended slab as FASTRS_TILE_RECORD_WORDS (20) u32 per
 *                       tile (count, max D, nfg, 0, 32 u16 counts of the entries with D bucket >= 4k)
 *                       plus the tiles' kept centres (uint2 each, tile
 *                       order; *n_entries <- their number, a device u64); unpack writes them into
 *                       the same layers of the receiver's workspace (its own layer indices)
 *   fastrs_slab_dilate  K5 on the own tiles from the tile data in the workspace
 * Together they give the same integer partials as fastrs_slab_reduce (K4's outputs for a tile
 * depend only on D within 3 slices of it).  All enqueue on `stream`; prune and dilate synchronise
 * once unless FASTRS_ASYNC. */
FASTRS_API int fastrs_slab_prune(const uint32_t* d_ext, const int64_t* dims_ext, int64_t own_lo, int64_t own_hi,
                                 uint32_t flags, void* ws, size_t ws_bytes, void* stream);
FASTRS_API int fastrs_slab_pack_tiles(void* ws, const int64_t* dims_ext, int64_t tz_a, int64_t tz_b, uint32_t* rec_out,
                                      void* ent_out, uint64_t* n_entries, void* stream);
FASTRS_API int fastrs_slab_unpack_tiles(void* ws, const int64_t* dims_ext, int64_t tz_a, int64_t tz_b,
                                        const uint32_t* rec_in, const void* ent_in, void* stream);
FASTRS_API int fastrs_slab_dilate(const int32_t* labels, const uint32_t* d_ext, const int64_t* dims_ext, int64_t own_lo,
                                  int64_t own_hi, int64_t Z, uint32_t dmax_global, int32_t max_label, uint32_t flags,
                                  uint64_t* vol, uint64_t* n_shell, uint64_t* sum_lt, uint64_t* sum_shell_lt,
                                  uint32_t* max_lt2, void* ws, size_t ws_bytes, void* stream);

/* D: closed forms from (reduced) partials: n_labels entries, nscale = elements per item used
 * for the fixed-point scale, dmax_global as in C.  Outputs as fastrs_sphericity_roundness. */
FASTRS_API int fastrs_metrics_from_partials(const uint64_t* vol, const uint64_t* n_shell, const uint64_t* sum_lt,
                                            const uint64_t* sum_shell_lt, const uint32_t* max_lt2,
                                            int64_t n_labels, int ndim, int64_t nscale, uint32_t dmax_global,
                                            double* sphericity, double* roundness,
                                            const fastrs_object_stats* stats, void* ws, size_t ws_bytes,
                                            void* stream);

/* ---- object filters of the paper's analysis protocol (label level) ----
 * fastrs_touches_edge: touches_edge[b*max_label + label-1] = 1 if some element of that label
 * lies on the boundary of its grid item (any face in 3D, any edge in 2D), else 0 (PAPER.md:195
 * "Edge cells are removed"; SPEC.md:212 remove_edge_objects).  labels as in
 * fastrs_sphericity_roundness (device); touches_edge: device, batch*max_label bytes, written in
 * full.  Labels outside 1..max_label are ignored.  FASTRS_EDGE_SKIP_ZLO / _ZHI leave out the first /
 * last z slice (a z-slab's inner faces; the slab path ORs the slabs' flags).  Errors: EINVAL
 * (geometry, NULL, max_label < 1), ECUDA.  Synchronises `stream` at the end unless FASTRS_ASYNC.
 * fastrs_filter_objects: sets sphericity[i] and roundness[i] (either may be NULL) to NaN where
 * volume[i] < min_volume ("the smallest objects are filtered out (V < 10^3)";
 * SPEC.md:219 filter_small) when volume != NULL, or where touches_edge[i] != 0 when touches_edge
 * != NULL; n_labels entries, all device pointers (volume: the stats output of
 * fastrs_sphericity_roundness).  Errors: EINVAL (n_labels < 0), ECUDA. */
FASTRS_API int fastrs_touches_edge(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                                   int32_t max_label, uint8_t* touches_edge, uint32_t flags, void* stream);
FASTRS_API int fastrs_filter_objects(double* sphericity, double* roundness, const int64_t* volume,
                                     const uint8_t* touches_edge, int64_t n_labels, int64_t min_volume,
                                     uint32_t flags, void* stream);

/* ---- multi-GPU z-slab call with NCCL inside the library -------
 * One process per GPU; rank r holds the z-slab [z0, z0 + nz) = fastrs_slab_partition(Z, P)[r]
 * (boundaries on multiples of 8 slices) of one 3D volume [Z][Y][X].  NCCL is loaded at run time
 * (dlopen of libnccl.so.2: the copy already mapped into the process, e.g. torch's, else the
 * system's; FASTRS_NCCL_LIB overrides), so the library itself loads without NCCL.
 *
 * fastrs_nccl_unique_id: 128-byte ncclUniqueId into id_out (rank 0; the caller broadcasts it).
 * fastrs_comm_init: *comm_out <- a communicator of nranks ranks on the current device
 *   (ncclCommInitRank; collective over the ranks); fastrs_comm_destroy frees it.
 * fastrs_slab_partition: bounds[0..nranks] of the z-slabs (the rule of slab.py: round(Z*i/P/8)*8).
 * fastrs_slab_halo_plan: the transfers that give every rank the w slices on each side of its
 *   slab: n_out entries (src, dst, side 0 lo / 1 hi, a, b), global slices [a, b); up to cap
 *   written to entries (5 int64 each; NULL: count only).  Pure host code.
 * fastrs_slab_call_workspace_bytes: device workspace of one fastrs_sphericity_roundness_slab
 *   call of this rank with halos of up to halo_cap slices (flags: FASTRS_SLAB_TRANSPOSE).
 * fastrs_sphericity_roundness_slab: collective over the communicator.  labels: the rank's slab
 *   [nz][Y][X] (device), dims_slab = {nz, Y, X}.  Exchanges (NCCL, on `stream`): the label slice
 *   below the slab; the z pass by an h-slice halo of packed EDT words, h = ceil(sqrt(max D_xy))
 *   (N8, default), or by the all-to-all z-slab <-> y-slab transpose (N1, FASTRS_SLAB_TRANSPOSE);
 *   the dilation halo, H = isqrt(Dmax - 1) rounded up to 8: by default the K4 outputs (tile records +
 *   kept centres) of the tile layers within H slices of each neighbour's slab, after a 3-slice D
 *   halo for K4's stencil (N4); with FASTRS_SLAB_DENSE_HALO the H slices of D; allreduce(sum)
 *   of the per-label u64 partial sums and allreduce(max) of max LT^2.  Every rank receives all
 *   max_label results (sphericity, roundness, stats: device, nullable), bit-identical to
 *   fastrs_sphericity_roundness on the whole volume.  info (host, nullable) reports the mode,
 *   the halo widths and the bytes this rank sent / received.  Errors as
 *   fastrs_sphericity_roundness, plus ENOMEM when h (N8) or H exceeds halo_cap (retry with a
 *   larger halo_cap and workspace), ENCCL on an NCCL failure.  Synchronises `stream` (twice, to
 *   size the halos). */
typedef struct {
  int32_t mode;              /* 0: N8 halo z pass, 1: N1 transpose                */
  int64_t h, H;              /* halo slices of the z pass (N8) and of the dilation */
  uint32_t dxy_max, dmax;    /* global max D_xy and max D                          */
  uint64_t bytes_sent, bytes_received;  /* exchanged by this rank (all phases)     */
} fastrs_slab_info;

FASTRS_API int fastrs_nccl_available(void);
FASTRS_API int fastrs_nccl_unique_id(void* id_out);
FASTRS_API int fastrs_comm_init(const void* id, int nranks, int rank, void** comm_out);
FASTRS_API int fastrs_comm_destroy(void* comm);
FASTRS_API int fastrs_slab_partition(int64_t Z, int nranks, int64_t* bounds);
FASTRS_API int fastrs_slab_halo_plan(const int64_t* bounds, int nranks, int64_t w, int64_t Z, int64_t* entries,
                                     int64_t cap, int64_t* n_out);
FASTRS_API int fastrs_slab_call_workspace_bytes(const int64_t* dims_slab, int64_t z0, int64_t Z, int nranks, int rank,
                                                int32_t max_label, int64_t halo_cap, uint32_t flags, size_t* bytes);
FASTRS_API int fastrs_sphericity_roundness_slab(const int32_t* labels, const int64_t* dims_slab, int64_t z0, int64_t Z,
                                                int32_t max_label, uint32_t flags, int64_t halo_cap,
                                                double* sphericity, double* roundness,
                                                const fastrs_object_stats* stats, fastrs_slab_info* info, void* comm,
                                                void* ws, size_t ws_bytes, void* stream);

/* ---- analysis protocol around the hot path --------------
 * fastrs_label_components: connected components of a binary mask (uint8 [batch][Z][Y][X],
 *   nonzero = object; "segmenting and labeling each fat component"):
 *   labels_out (int32, same shape, device) <- 0 on background, 1..K per item in the order of
 *   first encounter in a row-major scan (union-find whose roots are the smallest index of their
 *   component: canonical and deterministic); counts_out (device, batch int64, nullable) <- K.
 *   connectivity 4 / 8 (2D), 6 / 18 / 26 (3D).  Items below 2^32 elements.  Workspace:
 *   fastrs_ccl_workspace_bytes.  EINVAL on bad geometry / connectivity.  Synchronises.
 * fastrs_sphericity_wl: Eq. 3 width/length sphericity S = d2/d1 per label of a
 *   2D label image, d1 >= d2 = 4 sqrt(eigenvalues) of the label's pixel-coordinate covariance
 *   (population; the reading of SPEC.md:355-361, exact axes for a continuum ellipse); a single
 *   pixel gives 1.  Moments are exact integers.  swl, d1, d2: batch*max_label doubles (device,
 *   nullable), NaN for absent labels.  Workspace: fastrs_wl_workspace_bytes.  Synchronises.
 * fastrs_mc_measure: the S_MC baseline of PAPER.md:211/274 -- per label the iso-0.5 perimeter
 *   (2D marching squares, edge-midpoint crossings) or surface area (3D marching cubes: per-face
 *   midpoint segments, two diagonal inside corners cut separately, face segments closed into
 *   loops, each loop a centroid fan of triangles; reading r3) of the label's binary
 *   mask, the grid's outside counting as background; sphericity_mc = Eq. 2 (P_c / perimeter) in
 *   2D, Eq. 1 with the measured area in 3D.  Fixed-point per-label sums (bit-identical across
 *   runs).  measure, sphericity_mc: batch*max_label doubles (device, nullable).  Workspace:
 *   fastrs_mc_workspace_bytes.  Synchronises. */
FASTRS_API int fastrs_ccl_workspace_bytes(const int64_t* dims, int ndim, int64_t batch, size_t* bytes);
FASTRS_API int fastrs_label_components(const uint8_t* mask, const int64_t* dims, int ndim, int64_t batch,
                                       int connectivity, int32_t* labels_out, int64_t* counts_out, void* ws,
                                       size_t ws_bytes, void* stream);
FASTRS_API int fastrs_wl_workspace_bytes(int64_t batch, int32_t max_label, size_t* bytes);
FASTRS_API int fastrs_sphericity_wl(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                                    int32_t max_label, double* swl, double* d1, double* d2, void* ws, size_t ws_bytes,
                                    void* stream);
FASTRS_API int fastrs_mc_workspace_bytes(int64_t batch, int32_t max_label, size_t* bytes);
FASTRS_API int fastrs_mc_measure(const int32_t* labels, const int64_t* dims, int ndim, int64_t batch,
                                 int32_t max_label, double* measure, double* sphericity_mc, void* ws, size_t ws_bytes,
                                 void* stream);

FASTRS_API const char* fastrs_last_error(void);  /* thread-local message of the last failure */
FASTRS_API void fastrs_release(void);            /* free the per-device caches                */

#ifdef __cplusplus
}
#endif
#endif /* FASTRS_H */
