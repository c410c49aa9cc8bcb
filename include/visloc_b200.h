/*
 * visloc_b200 — C ABI of the B200-native LO-RANSAC PnP hot path.
 *
 * Drop-in boundary for the reference package `visloc` (pure Python/numpy,
 * /root/reference/pkg/src/visloc).  The reference has no native FFI: its
 * "operator API" is the set of module-level functions listed below, and a
 * drop-in is installed by rebinding them.  Each entry point
 * cites the reference function it replaces.
 *
 * Conventions
 *  - Every call returns an int status (VL_OK == 0).  Non-convergence of the
 *    estimator is NOT an error: it is reported in-band (converged = 0),
 *    exactly like PoseEstimate.converged (posest.py:278-289).
 *  - Large arrays are caller-owned DEVICE pointers (C-contiguous, fp64,
 *    row-major AoS exactly like the reference's numpy arrays: px (n,2),
 *    X (n,3), w (n)).  Small per-query metadata is passed in host memory.
 *  - All work is stream-ordered on the caller's cudaStream_t (passed as
 *    void*); calls that return host-visible scalars synchronise that stream.
 *  - A context is bound to one device and is not thread-safe; use one
 *    context per host thread / per GPU (one process per GPU is the model).
 *  - Workspace is library-owned and grows only in vl_reserve / on the first
 *    call that needs more; steady-state calls do not allocate.
 */
#ifndef VISLOC_B200_H
#define VISLOC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  VL_OK = 0,
  VL_ERR_INVALID = 1,          /* bad argument -> ValueError */
  VL_ERR_CUDA = 2,             /* CUDA runtime error */
  VL_ERR_OOM = 3,              /* device allocation failed */
  VL_ERR_UNDERCONSTRAINED = 4, /* n < 3 -> UnderConstrainedError (posest.py:232-234) */
  VL_ERR_SINGULAR = 5          /* refine with < 3 points (refine.py:185-186) */
};

typedef struct vl_ctx vl_ctx;

/* Pinhole intrinsics (geometry.py:44-76); width/height are not needed on device. */
typedef struct { double fx, fy, cx, cy; } vl_intrinsics;

/* numpy PCG64 bit-generator state (numpy 2.3.5 `bit_generator.state`):
 * 128-bit state and increment split in 64-bit halves + the uint32 buffer. */
typedef struct {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
  uint32_t has_uint32, uinteger;
} vl_pcg64_state;

/* RansacConfig (posest.py:69-90).  cauchy_scale <= 0 means "None -> tau". */
typedef struct {
  int64_t max_iterations;
  int32_t batch_size;
  int32_t max_scoring;
  double miss_probability;
  double reproj_threshold;
  double cauchy_scale;
  int32_t lm_max_iters;
  int32_t _pad;
} vl_ransac_config;

/* Batched ransac_pnp (posest.py:223-299): Q independent queries whose
 * matches are concatenated; query i owns rows [offsets[i], offsets[i+1]). */
typedef struct {
  int32_t num_queries;
  int32_t _pad;
  const int64_t* offsets;      /* HOST [Q+1] */
  const vl_intrinsics* intr;   /* HOST [Q] */
  const vl_pcg64_state* rng;   /* HOST [Q] initial generator state (default_rng(seed)) */
  const double* px;            /* DEVICE [N,2] query pixels */
  const double* X;             /* DEVICE [N,3] world points */
  const double* w;             /* DEVICE [N]  confidence weights (> 0) */
  vl_ransac_config cfg;
} vl_ransac_args;

/* PoseEstimate (posest.py:93-103), one row per query; all DEVICE pointers. */
typedef struct {
  double* q;                /* [Q,4] scalar-first unit quaternion, w >= 0 */
  double* t;                /* [Q,3] */
  uint8_t* inlier_flags;    /* [N]   */
  int64_t* inlier_count;    /* [Q]   */
  double* score;            /* [Q]   fp64 MSAC cost of the final pose (inf on failure) */
  int64_t* iterations;      /* [Q]   minimal samples drawn */
  int32_t* converged;       /* [Q]   */
  int64_t* stats;           /* [Q,4] optional (may be NULL): lo_calls, hypotheses, evals, rounds */
} vl_ransac_out;

/* ---- context ---------------------------------------------------------- */
int vl_create(int device, vl_ctx** out);
int vl_destroy(vl_ctx* ctx);
const char* vl_last_error(vl_ctx* ctx);
/* Pre-size the workspace (optional). */
int vl_reserve(vl_ctx* ctx, int32_t max_queries, int64_t max_n_per_query, int32_t batch_size);
/* Number of kernel launches issued by this context since creation. */
int64_t vl_launch_count(vl_ctx* ctx);

/* Profiling: when enabled, every stage launch of vl_ransac_pnp is bracketed
 * by CUDA events on the caller's stream and accumulated per stage (order:
 * prep, sample, p3p, compact, score, scan, active, final).  Enabling resets. */
int vl_profile(vl_ctx* ctx, int enable);
int vl_profile_read(vl_ctx* ctx, double* ms, int64_t* launches, int32_t n);

/* Exact scoring pruning (default on; env VISLOC_PRUNE=0 turns it off for a
 * context that never called this).  In rounds with a best pose, the fp32
 * MSAC sum of a hypothesis (posest.py:178-220) is first formed over a prefix
 * of the scoring subset; the terms are non-negative and fp32 addition is
 * monotone, so a prefix >= the best cost proves that the ordered scan
 * (`costs[h] < best_cost`, posest.py:258) rejects the hypothesis, and only
 * the others are scored to the end.  Every output is identical either way;
 * only the number of evaluations executed changes.  Queries with a negative
 * weight are never pruned. */
int vl_set_scoring_pruning(vl_ctx* ctx, int32_t enable);
/* Run totals since the last reset: out[0] = hypothesis x correspondence
 * evaluations skipped by pruning, out[1] = evaluations done by the tail pass
 * for the hypotheses that survived the prefix.  Synchronises the device. */
int vl_scoring_counters(vl_ctx* ctx, int64_t* out, int32_t reset);

/* numpy SeedSequence(seed) -> PCG64 state (np.random.default_rng(seed),
 * posest.py:243).  Host-only helper, no device work. */
int vl_pcg64_seed(uint64_t seed, vl_pcg64_state* out);

/* ---- hot path ---------------------------------------------------------- */
/* replaces visloc.posest.ransac_pnp (posest.py:223) — batched over queries */
int vl_ransac_pnp(vl_ctx* ctx, const vl_ransac_args* args, const vl_ransac_out* out, void* stream);

/* Same estimator with staged admission, for callers that stream the inputs
 * to the device: the rows of stage k (queries [stage_end[k-1], stage_end[k]),
 * stage_end HOST [nstage], last = num_queries) are read only after
 * stage_events[k] (a cudaEvent_t recorded after that stage's host-to-device
 * copy, on any stream) has completed.  All stages share one round loop, so
 * later copies overlap the rounds of admitted queries.  Results equal
 * vl_ransac_pnp's.  A run larger than one workspace chunk (4096 queries at
 * batch_size 1000, fewer for larger batches) runs its chunks in order, each
 * admitting the stages that overlap it. */
int vl_ransac_pnp_staged(vl_ctx* ctx, const vl_ransac_args* args, const vl_ransac_out* out, int32_t nstage,
                         const int32_t* stage_end, void* const* stage_events, void* stream);

/* Stepwise driver of the same estimator, for the optional single-query
 * hypothesis-split mode across GPUs.  Every rank calls
 * vl_ransac_begin with identical args and its (split_rank, split_size):
 * samples, P3P and scans are replicated, the scoring tiles (query, 256 or
 * 768 hypotheses) are dealt round-robin and non-owned tiles hold zero costs.
 * Per round:
 *   vl_ransac_step_score(ctx, buf)      -> this rank's fp32 cost vector [Q][HCAP] into buf (DEVICE)
 *   SUM all-reduce of buf across ranks  (NCCL over NVLink; exact: one non-zero term;
 *                                        vl_ransac_partial_bytes = 4*Q*HCAP, 16 KB/query at B=1000)
 *   vl_ransac_step_finish(ctx, buf, &n) -> ordered scan / LO / stop; n active queries
 * until n == 0, then vl_ransac_end(ctx, out).  Results are bit-identical on
 * every rank and to vl_ransac_pnp.  One workspace chunk of queries. */
int vl_ransac_begin(vl_ctx* ctx, const vl_ransac_args* args, int32_t split_rank, int32_t split_size,
                    void* stream);
int vl_ransac_partial_bytes(vl_ctx* ctx, int64_t* bytes);
int vl_ransac_step_score(vl_ctx* ctx, void* partial_out, void* stream);
int vl_ransac_step_finish(vl_ctx* ctx, const void* partial_in, int32_t* nactive, void* stream);
int vl_ransac_end(vl_ctx* ctx, const vl_ransac_out* out, void* stream);
/* BASELINE's packed (score, index) variant of the hypothesis split — an
 * APPROXIMATION of the reference (at most one LO per round, on the batch's
 * best hypothesis, instead of the ordered first-better chain).  Per round:
 *   vl_ransac_step_score(ctx, NULL)        -> this rank's owned costs
 *   vl_ransac_step_argmin(ctx, keys)       -> keys DEVICE int64 [Q]: min over owned
 *                                             hypotheses of float_bits(cost) << 32 | h
 *   MIN all-reduce of keys across ranks    (8 B per query)
 *   vl_ransac_step_finish_argmin(ctx, keys, &n) -> scan / LO / stop on the winner */
int vl_ransac_step_argmin(vl_ctx* ctx, int64_t* keys, void* stream);
int vl_ransac_step_finish_argmin(vl_ctx* ctx, const int64_t* keys, int32_t* nactive, void* stream);

/* replaces visloc.posest.msac_score (posest.py:160).  pose q[4], t[3] HOST;
 * arrays DEVICE; cost -> *cost_out (HOST), flags -> DEVICE (may be NULL). */
int vl_msac_score(vl_ctx* ctx, const double* q, const double* t, const double* px,
                  const double* X, const double* w, int64_t n, vl_intrinsics intr, double tau,
                  double* cost_out, uint8_t* flags, void* stream);

/* replaces visloc.posest._score_hypotheses (posest.py:178-220): the fp32
 * ranking costs of H hypotheses (R DEVICE [H,3,3] row-major, t DEVICE [H,3])
 * against one scoring set (px/X/w DEVICE, n rows) through the estimator's own
 * k_score kernel (records, fx/fy-folded rows, canonical split sums).
 * shape: 0 = the estimator's single-query tiles, 1 = fine, 2 = coarse tiles
 * (same bits by construction).  costs DEVICE [H] f32.  Uses the context's
 * estimator workspace: VL_ERR_INVALID while a stepwise run is open. */
int vl_score_hypotheses(vl_ctx* ctx, const double* R, const double* t, int32_t H, const double* px,
                        const double* X, const double* w, int64_t n, vl_intrinsics intr, double tau,
                        int32_t shape, float* costs, void* stream);

/* replaces visloc.refine.refine_pose (refine.py:164).  loss: 0 truncated
 * (TruncatedLoss(scale)), 1 Cauchy (CauchyLoss(scale)).  q_io/t_io HOST
 * in/out; trace HOST [max_iters+1] (may be NULL). */
int vl_refine_pose(vl_ctx* ctx, double* q_io, double* t_io, const double* px, const double* X,
                   const double* w, int64_t n, vl_intrinsics intr, int32_t loss, double scale,
                   int32_t max_iters, double gradient_tol, double cost_tol, int32_t* converged,
                   int32_t* iterations, double* trace, int32_t* trace_len, void* stream);

/* replaces visloc.refine.robust_cost (refine.py:135-149): pose q/t HOST,
 * arrays DEVICE, *cost_out HOST (inf for Cauchy with a point behind). */
int vl_robust_cost(vl_ctx* ctx, const double* q, const double* t, const double* px, const double* X,
                   const double* w, int64_t n, vl_intrinsics intr, int32_t loss, double scale,
                   double* cost_out, void* stream);

/* replaces visloc.refine.pose_residuals + pose_jacobian (refine.py:90-132):
 * res DEVICE [n,2], z DEVICE [n], J DEVICE [n,2,6] (each may be NULL). */
int vl_pose_residuals(vl_ctx* ctx, const double* q, const double* t, const double* px, const double* X,
                      int64_t n, vl_intrinsics intr, double* res, double* z, double* J, void* stream);

/* replaces visloc.p3p.p3p_solve_batch (p3p.py:57).  bearings/points DEVICE
 * [B,3,3]; outputs DEVICE R [4B,3,3], t [4B,3], sample [4B]; *m_out HOST. */
int vl_p3p_solve_batch(vl_ctx* ctx, const double* bearings, const double* points, int32_t B,
                       double* R, double* t, int64_t* sample, int32_t* m_out, void* stream);

/* Reproduce numpy's `rng.choice(n, 3, replace=False)` stream on device
 * (posest.py:252): `count` samples from state `st` (HOST), written to DEVICE
 * out [count,3] (int32; n < 2^31 on the path); the advanced generator state
 * is written back to *st (HOST), matching numpy's `bit_generator.state`. */
int vl_sample_minimal_sets(vl_ctx* ctx, vl_pcg64_state* st, int64_t n, int32_t count,
                           int32_t* out, void* stream);

/* ---- retrieval (retrieval.DescriptorIndex.topk, retrieval.py:66-82) ----- */
/* Exact cosine top-k for Q queries at once.  db DEVICE [E,D] fp64 rows, unit
 * normalised as DescriptorIndex.add stores them (f32 rows widened); id_rank
 * DEVICE [E] = position of each entry id in ascending id order (the tie
 * key); queries DEVICE [Q,D] fp64, normalised here; 1 <= k <= 32.  out_idx
 * DEVICE [Q, min(k,E)] entry rows best first (similarity descending, ties by
 * ascending id), out_sim DEVICE [Q, min(k,E)].  A zero or non-finite query
 * -> VL_ERR_INVALID ("query vector must be non-zero and finite"). */
int vl_retrieval_topk(vl_ctx* ctx, const double* db, const int64_t* id_rank, int32_t E, int32_t D,
                      const double* queries, int32_t Q, int32_t k, int32_t* out_idx, double* out_sim,
                      void* stream);

/* ---- IMLC correspondence-field files (matchio.py:9-20, read_field :158-200) */
enum {
  VL_IMLC_OK = 0,
  VL_IMLC_MAGIC = 1,     /* FieldMagicError, offset 0 */
  VL_IMLC_VERSION = 2,   /* FieldVersionError, offset 4 */
  VL_IMLC_TRUNCATED = 3, /* FieldTruncatedError: need `need` bytes for `what`, have `have` */
  VL_IMLC_TRAILING = 4   /* FieldFormatError: `have` trailing bytes after the records */
};

/* Parsed header of one little-endian IMLC blob.  Byte ranges are relative to
 * the blob start; records are grid_h*grid_w x (target_x f32, target_y f32,
 * conf f32), row-major, starting at records_off (not necessarily aligned). */
typedef struct {
  int32_t status;         /* VL_IMLC_* */
  uint32_t version;       /* as read (VL_IMLC_VERSION reports it) */
  int64_t error_offset;   /* FieldFormatError.offset */
  int64_t need, have;     /* truncation / trailing-byte details */
  const char* what;       /* static string: the field being read when truncated */
  uint8_t magic[4];       /* as read (VL_IMLC_MAGIC reports it) */
  uint32_t grid_w, grid_h;
  double scale_x, scale_y;
  int64_t source_off, source_len, target_off, target_len;
  int64_t records_off;
} vl_imlc_header;

/* Host-only header parse with read_field's validation order and error
 * offsets (matchio.py:160-190).  Returns VL_OK when the call itself worked
 * (the blob's verdict is out->status), VL_ERR_INVALID on null arguments.
 * Record CONTENT (confidence finite in [0,1], finite targets where conf > 0;
 * matchio.py:99-109) is validated on the GPU by vl_lift (VL_LIFT_IMLC). */
int vl_imlc_parse(const uint8_t* blob, int64_t len, vl_imlc_header* out);

/* ---- depth lifting (localizer.lift, localizer.py:134-197) -------------- */
/* One correspondence field, in output order (entry id, then db->query
 * (direction 0, direct depth lookup) before query->db (direction 1,
 * bilinear depth)).  layout VL_LIFT_PLANAR: targets (gh,gw,2) and confidence
 * (gh,gw) arrays in f32 (file-backed) or f64 (in-memory) — one dtype per
 * call (field_f64).  layout VL_LIFT_IMLC: `targets` points at the IMLC
 * records (12-byte (x, y, conf) f32 triples, 4-byte aligned), `confidence`
 * is ignored; the records may live in HBM or in mapped pinned host memory.
 * Arrays are DEVICE-accessible pointers. */
enum { VL_LIFT_PLANAR = 0, VL_LIFT_IMLC = 1 };
typedef struct {
  int32_t query, entry, direction, depth; /* depth: index into the vl_lift_depth array */
  int32_t grid_w, grid_h;
  int32_t layout, _pad;
  double scale_x, scale_y;                /* cell -> pixel (matchio.py:83-84) */
  const void* targets;
  const void* confidence;
} vl_lift_segment;

/* Per-segment content verdict of VL_LIFT_IMLC segments (vl_lift seg_flags):
 * the first violated rule in CorrespondenceField.__post_init__ order. */
enum { VL_FIELD_BAD_CONF = 1, VL_FIELD_BAD_TARGET = 2 };

/* A database entry's stored depth + camera.  kind: 0 f32 values + valid,
 * 1 f16 values + valid, 2 u8 log codes, 3 u16 log codes (code 0 invalid;
 * `lut` = dequantize_depth table, mapstore.py:122-134). */
typedef struct {
  int32_t width, height, kind, _pad;
  const void* values;                     /* DEVICE [h,w] */
  const uint8_t* valid;                   /* DEVICE [h,w] (kinds 0, 1) */
  const float* lut;                       /* DEVICE [levels+1] (kinds 2, 3) */
  double fx, fy, cx, cy;                  /* database intrinsics */
  double sx_depth, sy_depth;              /* depth width / image width, depth height / image height */
  double R[9], t[3];                      /* database pose, camera-from-world */
} vl_lift_depth;

/* replaces localizer.lift for many (query, entry) field pairs at once;
 * mode 0 = lift, mode 1 = confidence gate only (matchio.filter_matches_arrays,
 * outputs px = source px, X = (target x, target y, flat cell index)).
 * Outputs DEVICE (capacity rows); seg_offsets HOST [nseg+1] receives the
 * exclusive output offset of every segment (last = total matches);
 * seg_flags HOST [nseg] (nullable) receives the VL_FIELD_* content verdict
 * of every IMLC segment (0 = valid; always 0 for planar segments);
 * entry_out DEVICE (nullable): the segment's `entry` index per output row. */
int vl_lift(vl_ctx* ctx, const vl_lift_segment* segs, int32_t nseg, const vl_lift_depth* depths,
            int32_t ndepth, int32_t field_f64, double threshold, int32_t mode, double* px_out,
            double* X_out, double* w_out, int32_t* entry_out, int64_t capacity, int64_t* seg_offsets,
            int32_t* seg_flags, void* stream);

/* replaces localizer.interp_depth_many (localizer.py:87-115): pts DEVICE
 * [n,2] depth-map subpixels; vals DEVICE [n] (0 where invalid), ok DEVICE [n]. */
int vl_interp_depth(vl_ctx* ctx, const vl_lift_depth* depth, const double* pts, int64_t n, double* vals,
                    uint8_t* ok, void* stream);

/* replaces mapstore.dequantize_depth (mapstore.py:122-134) applied on device:
 * codes (kinds 2, 3) -> f32 depth (0 where invalid) + valid. */
int vl_decode_depth(vl_ctx* ctx, const vl_lift_depth* depth, float* vals, uint8_t* valid, void* stream);

/* ---- depth-map codecs (mapstore.py:96-134, :390-425) --------------------- */
/* One depth map.  quantize: kind 0 (f32 values) or 1 (f16 values) + valid
 * (u8) in, codes out (u8 when levels <= 255, else u16).  reduce: kind 2 (u8
 * codes) or 3 (u16 codes) with `levels` in, codes of the new level count out
 * ((h+f-1)/f x (w+f-1)/f, u8 when new_levels <= 255, else u16).  All arrays
 * DEVICE, row-major [h,w]. */
typedef struct {
  int32_t width, height, kind, levels;
  const void* values;
  const uint8_t* valid;
  void* out;
} vl_depth_codec_job;

/* replaces mapstore.quantize_depth (mapstore.py:96-119) for many maps:
 * `thresholds` DEVICE [levels-1] ascending f32 — entry k is the smallest f32
 * depth the reference maps to code k+2 (built on the host with the reference's
 * own fp64 arithmetic); a valid pixel's code is 1 + #{thresholds <= depth},
 * invalid pixels get 0. */
int vl_quantize_depth(vl_ctx* ctx, const vl_depth_codec_job* jobs, int32_t njobs, const float* thresholds,
                      int32_t levels, void* stream);

/* replaces mapstore._downsample_codes_nearest_valid + _requantize_codes
 * (mapstore.py:390-425; reduce_map's depth step, :428-497) for many maps:
 * block factor >= 1, new_levels in [1, 65535]. */
int vl_reduce_depth_codes(vl_ctx* ctx, const vl_depth_codec_job* jobs, int32_t njobs, int32_t factor,
                          int32_t new_levels, void* stream);

/* ---- dense depth triangulation (depthbuild.py:104-441) ------------------ */
/* A covisible view of a map being triangulated: the planar correspondence
 * field from the map's entry to this view (DEVICE targets (gh,gw,2) and
 * confidence (gh,gw); f32 or f64, one dtype per call) and the view's camera. */
typedef struct {
  const void* targets;
  const void* confidence;
  double rt[9];                /* R^T of the view pose (world-from-camera rotation), row-major */
  double center[3];            /* view camera centre (Pose.center()) */
  double fx, fy, cx, cy;       /* view intrinsics */
} vl_tri_view;

/* One depth map to build: views [view0, view0+nview) of the view array. */
typedef struct {
  int32_t grid_w, grid_h, view0, nview;
  double fx, fy, cx, cy;       /* entry intrinsics (full image) */
  double sx, sy;               /* width / grid_w, height / grid_h (depthbuild.py:312-313) */
  double R[9];                 /* entry pose rotation (camera-from-world), row-major */
  double center[3];            /* entry camera centre */
  float* depth;                /* DEVICE (gh,gw) z-depth out (0 where invalid) */
  uint8_t* valid;              /* DEVICE (gh,gw) out */
} vl_tri_map;

/* TriangulationConfig (depthbuild.py:80-93) */
typedef struct {
  double angular_threshold_rad, confidence_threshold, refine_tol;
  int32_t min_inliers, max_refine_iters;
} vl_tri_config;

/* replaces depthbuild.build_depth_map (depthbuild.py:249-375) for many maps in
 * one launch; maps / views are HOST arrays (copied by the call), nview <= 128
 * per map.  Returns after the maps are written (stream synchronised). */
int vl_build_depth_maps(vl_ctx* ctx, const vl_tri_map* maps, int32_t nmap, const vl_tri_view* views,
                        int32_t nviews, int32_t field_f64, const vl_tri_config* cfg, void* stream);

/* An explicit observation set (triangulate_pixel's arguments, depthbuild.py:151-189). */
typedef struct {
  double ray[3], center[3];    /* unit reference ray (world) and reference centre */
  int32_t obs0, nobs;          /* observations [obs0, obs0+nobs) */
} vl_tri_problem;

typedef struct {
  double rt[9], center[3];     /* observing view: R^T, centre */
  double fx, fy, cx, cy;
  double target[2];            /* matched pixel in the observing view */
  double confidence;
} vl_tri_obs;

/* replaces depthbuild.triangulate_pixel / depth_hypothesis (depthbuild.py:104-189)
 * for many problems: problems / obs DEVICE; depth_out DEVICE [nprob] (ray
 * depth, NaN if none), count_out DEVICE [nprob] (winning inlier count, 0 if
 * none), hyp_out DEVICE [total obs] nullable (each observation's depth
 * hypothesis, NaN where depth_hypothesis returns None). max_obs <= 128. */
int vl_triangulate_rays(vl_ctx* ctx, const vl_tri_problem* problems, int32_t nprob, const vl_tri_obs* obs,
                        int32_t max_obs, const vl_tri_config* cfg, double* depth_out, int32_t* count_out,
                        double* hyp_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* VISLOC_B200_H */
