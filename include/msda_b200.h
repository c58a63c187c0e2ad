/*
 * msda_b200 — C ABI of the B200-native Multi-Scale Deformable Aggregation path.
 *
 * Drop-in boundary for the reference operator (paths relative to
 * /root/reference/pkg/src/mvtrack3d/):
 *
 *   msda_csr()       replaces msda_reference(pyramids, plan, normalize)      features.py:241-276
 *                    and      msda_optimized(pyramids, plan, precision,
 *                                            normalize, workers)           features.py:419-467
 *   msda_dense()     the Sparse4D operator named by BASELINE north_star:
 *                    deformable_aggregation(mc_ms_feat, spatial_shape,
 *                    scale_start_index, sampling_location, weights); the
 *                    reference has no such symbol, its semantics here are the
 *                    reference's (zero padding, cell = loc*W - 0.5,
 *                    features.py:20-24, 184-219) with channel groups G.
 *   msda_dense_project()  msda_dense with keypoint generation + projection
 *                    fused in (geometry.py:162-182, 207-255; oae.py:103-111)
 *   msda_oae_pool()  extract_view_feature + fuse_or_memory (oae.py:81-164)
 *   msda_csr_host()  msda_csr over HOST buffers (what a ctypes binding of
 *                    mvtrack3d would call with numpy pointers); copies in and
 *                    out inside the call.
 *
 * Conventions: every pointer is a device pointer unless the entry point says
 * HOST.  The caller owns every buffer, the workspace and the stream; calls are
 * asynchronous on `stream` (a cudaStream_t passed as void*), never allocate
 * (except the context API) and keep no global state.  Argument errors are
 * returned synchronously; data-dependent errors (zero weight sum, unknown
 * camera/level, non-finite plan values) are written to a status word in the
 * workspace and read back with msda_read_status().
 */
#ifndef MSDA_B200_H_
#define MSDA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; each maps to the reference exception raised for it. */
enum msda_status {
  MSDA_OK = 0,
  MSDA_ODD_CHANNELS = 1,     /* errors.OddChannelCount   features.py:98-99, 441-442        */
  MSDA_NONFINITE = 2,        /* errors.NonFiniteWeight   features.py:165-166               */
  MSDA_BAD_TARGET = 3,       /* ValueError unknown camera / missing level  features.py:231-238 */
  MSDA_ZERO_WEIGHT_SUM = 4,  /* ValueError zero weight sum  features.py:268-269, 285-287   */
  MSDA_BAD_PRECISION = 5,    /* ValueError unknown precision mode  features.py:443-444     */
  MSDA_CHANNEL_MISMATCH = 6, /* errors.ChannelMismatch   oae.py:98-100                     */
  MSDA_CUDA_ERROR = 7,       /* CUDA runtime failure                                       */
  MSDA_BAD_ARG = 8,          /* shape / pointer / workspace argument error (ValueError)    */
  MSDA_OFFSET_RANGE = 9      /* errors.OffsetOutOfRange  geometry.py:241-243               */
};

/* Feature storage dtype. */
enum msda_dtype { MSDA_F32 = 0, MSDA_F16 = 1, MSDA_BF16 = 2 };

/* Arithmetic mode.
 *  MSDA_EXACT      f32 arithmetic in the reference's canonical order and
 *                  expression tree: bit-identical to msda_reference /
 *                  msda_optimized(FULL) (f32 storage) or to the reference run on
 *                  features pre-rounded to the storage dtype (f16/bf16).
 *  MSDA_EXACT_HALF f16 storage and f16 arithmetic/accumulation, bit-identical
 *                  to msda_optimized(PACKED_HALF) (features.py:306-416).
 *  MSDA_FAST       FMA arithmetic, any summation order, f32 accumulation;
 *                  tolerance parity (1e-4 rel. fp32, 1e-2 fp16/bf16).
 *  MSDA_FAST_H2    dense path, f16 storage: products and per-camera partial
 *                  sums in half2 (the paper's half2 accumulation), flushed to
 *                  f32 per camera; 1e-2 tolerance.  Other dtypes: = FAST.      */
enum msda_precision { MSDA_EXACT = 0, MSDA_EXACT_HALF = 1, MSDA_FAST = 2, MSDA_FAST_H2 = 3 };

/* Multi-camera multi-level feature table: channel-last rows, every
 * (camera, level) grid (H, W, C) row-major, concatenated camera-major then
 * level-minor.  `batch` copies of the table are stacked (stride n_rows*C).  */
typedef struct {
  const void *data;                 /* [batch, n_rows, channels]                      */
  int32_t dtype;                    /* enum msda_dtype                               */
  int32_t batch;                    /* >= 1                                          */
  int32_t n_cams, n_levels, channels;
  int32_t reserved;
  int64_t n_rows;                   /* < 2^31                                        */
  const int32_t *spatial_shape;     /* [n_cams * n_levels * 2] (H, W)                */
  const int64_t *scale_start_index; /* [n_cams * n_levels] first row of each grid    */
  const int32_t *spatial_shape_host; /* optional HOST copy of spatial_shape, or NULL:
                                        lets a call pick the on-chip staging plan
                                        without reading device memory (ABI v2)   */
} msda_features_t;

/* CSR sample plan (the reference SamplePlan, features.py:112-181).  Camera
 * ids are given as dense indices 0..n_cams-1 in ascending camera-id order.  */
typedef struct {
  int64_t n_queries, n_samples;
  const int64_t *offsets;      /* [n_queries + 1]                        */
  const int32_t *camera_index; /* [n_samples]                            */
  const int32_t *level;        /* [n_samples]                            */
  const float *u, *v;          /* [n_samples] level-cell coordinates     */
  const float *weight;         /* [n_samples]                            */
} msda_csr_plan_t;

/* Pinhole cameras (CameraModel, geometry.py:56-97), float64 on device (the
 * reference projects in f64; so does the fused kernel). */
typedef struct {
  const double *K;       /* [n_cams, 4]  fx, fy, cx, cy              */
  const double *R;       /* [n_cams, 9]  world->camera rotation      */
  const double *t;       /* [n_cams, 3]  world->camera translation   */
} msda_cameras_t;

const char *msda_status_string(int32_t status);
int32_t msda_abi_version(void);

/* Workspace: one device buffer sized by the matching *_workspace_size(). */
size_t msda_csr_workspace_size(int64_t n_queries, int64_t n_samples, int32_t channels);
int32_t msda_csr(const msda_features_t *feat, const msda_csr_plan_t *plan, int32_t precision,
                 int32_t normalize, float *out /* [n_queries, C] */, uint8_t *empty /* [n_queries] */,
                 void *workspace, size_t workspace_bytes, void *stream);

/* msda_csr split into its two stages (bit 0: canonicalise the plan into the
 * workspace, bit 1: gather/accumulate from the workspace); msda_csr == mask 3.
 * Used to time the stages separately.                                       */
int32_t msda_csr_stages(const msda_features_t *feat, const msda_csr_plan_t *plan, int32_t precision,
                        int32_t normalize, float *out, uint8_t *empty, void *workspace, size_t workspace_bytes,
                        void *stream, int32_t stage_mask);

size_t msda_dense_workspace_size(int32_t batch, int32_t n_queries, int32_t n_points, int32_t n_cams,
                                 int32_t n_levels, int32_t n_groups, int32_t channels);
/* sampling_location [bs, Q, P, cams, 2] normalized (x, y) in image units,
 * weights [bs, Q, P, cams, L, G], out [bs, Q, C].  Channel c uses group
 * c / (C / G).  normalize: divide by the per-(query, group) weight sum.     */
int32_t msda_dense(const msda_features_t *feat, int32_t n_queries, int32_t n_points, int32_t n_groups,
                   const float *sampling_location, const float *weights, int32_t precision,
                   int32_t normalize, float *out, void *workspace, size_t workspace_bytes, void *stream);

/* Camera-sharded partials (paper_2601_10819_b200/dist.py): FAST aggregation of
 * this rank's cameras without normalisation, plus the per-(query, group)
 * weight sums weight_sums [bs*Q, G]; after summing both across ranks (NCCL
 * all-reduce), msda_dense_normalize divides out by the sums (zero sum ->
 * MSDA_ZERO_WEIGHT_SUM in the workspace status word, msda_read_status).    */
int32_t msda_dense_partial(const msda_features_t *feat, int32_t n_queries, int32_t n_points, int32_t n_groups,
                           const float *sampling_location, const float *weights, int32_t precision, float *out,
                           float *weight_sums, void *workspace, size_t workspace_bytes, void *stream);
int32_t msda_dense_normalize(float *out, const float *weight_sums, int64_t n_queries, int32_t channels,
                             int32_t n_groups, void *workspace /* >= 256 B */, void *stream);

/* Camera-sharded all-reduce over peer memory (NVLink), the alternative to
 * msda_dense_partial -> NCCL all-reduce -> msda_dense_normalize: every rank
 * pushes its partial numerators [rows, C] and weight sums [rows, G] into
 * every rank's symmetric buffer (float4 red.add through CUDA-IPC mappings),
 * signals with a system-scope release counter, waits for all ranks and
 * writes out = num / wsum per group (normalize) or num.  Buffers:
 * msda_peer_alloc(msda_peer_buffer_size(rows, C, G)) on every rank, handles
 * exchanged with msda_ipc_handle / msda_ipc_open (64 bytes each);
 * peer_buffers[r] = rank r's buffer as mapped here (own buffer at [rank]).
 * epoch: 1, 2, 3, ... identical on every rank, one per call.  A rank that
 * never arrives makes the call report MSDA_CUDA_ERROR (status word) after a
 * bounded wait. */
/* Page-lock / release an existing host range (a memory-mapped FPYR payload:
 * frames then go to the device as one DMA each, no staging copy).
 * read_only != 0 for read-only mappings.  MSDA_CUDA_ERROR when the range
 * cannot be registered (the caller stages through a pinned buffer). */
int32_t msda_host_register(void *ptr, size_t bytes, int32_t read_only);
int32_t msda_host_unregister(void *ptr);

#define MSDA_IPC_HANDLE_BYTES 64
size_t msda_peer_buffer_size(int64_t rows, int32_t channels, int32_t groups);
int32_t msda_peer_alloc(size_t bytes, void **ptr);
int32_t msda_peer_free(void *ptr);
int32_t msda_ipc_handle(const void *ptr, void *handle /* MSDA_IPC_HANDLE_BYTES */);
int32_t msda_ipc_open(const void *handle, void **ptr);
int32_t msda_ipc_close(void *ptr);
int32_t msda_peer_allreduce_normalize(const float *num, const float *weight_sums, void *const *peer_buffers,
                                      int32_t world, int32_t rank, uint32_t epoch, int64_t rows, int32_t channels,
                                      int32_t groups, int32_t normalize, float *out, float *wsum_out,
                                      void *workspace /* >= 256 B */, void *stream);

/* Fused projection: anchors [bs, Q, 10] (x, y, z, w, l, h, yaw, vx, vy, vz),
 * learned_offsets [n_learned, 3] in [-1, 1], P = 7 + n_learned keypoints
 * (geometry.py:207-247), motion compensation by velocity*dt
 * (geometry.py:250-255), projection in f64 (geometry.py:162-182) with
 * behind-camera samples (depth <= 1e-6) dropped from the plan (weight and
 * contribution); cell = pixel / strides[level] - 0.5 (features.py:45-47).
 * weights [bs, Q, P, cams, L, G]; workspace = msda_dense_workspace_size(). */
int32_t msda_dense_project(const msda_features_t *feat, int32_t n_queries, const float *anchors,
                           int32_t n_learned, const float *learned_offsets, const msda_cameras_t *cams,
                           const float *strides, float dt, int32_t n_groups, const float *weights,
                           int32_t precision, int32_t normalize, float *out, void *workspace,
                           size_t workspace_bytes, void *stream);

/* OAE pooling (cfg4): per (query, camera) g = softmax_k(desc . g_k / sqrt(D))
 * weighted keypoint features (level mean), fused over cameras with
 * visibility weights (invalid views weigh 0), L2-normalised; queries whose
 * visibility sum is <= 1e-3 get `memory` and all_occluded = 1.
 * descriptors / memory [Q, D=C], visibility [Q, n_cams], out [Q, C].       */
int32_t msda_oae_pool(const msda_features_t *feat, int32_t n_queries, const float *anchors,
                      int32_t n_learned, const float *learned_offsets, const msda_cameras_t *cams,
                      const float *strides, const float *descriptors, const float *visibility,
                      const float *memory, float *out, uint8_t *all_occluded, void *workspace,
                      size_t workspace_bytes, void *stream);
size_t msda_oae_workspace_size(int32_t n_queries, int32_t n_cams, int32_t channels);

/* Visible fraction of every object in every camera (visibility.py:46-115):
 * objects [n_objects, 9] f64 (x, y, z, w, l, h, yaw, cos(yaw), sin(yaw)) with
 * cos / sin from the HOST libm (Python's math.cos / math.sin in rot_z,
 * geometry.py:50-53: the counts are then bit-exact), image_wh [n_cams, 2]
 * int32, grid samples per axis (reference default 64).  Out: visibility
 * [n_cams, n_objects] f32 in [0, 1], fully_behind [n_cams, n_objects] (no box
 * corner in front of the camera -> visibility 0).  These are the v_i that
 * msda_oae_pool consumes.                                                   */
size_t msda_visibility_workspace_size(int32_t n_cams, int32_t n_objects);
int32_t msda_visibility(const msda_cameras_t *cams, const int32_t *image_wh, int32_t n_cams,
                        const double *objects, int32_t n_objects, int32_t grid, float *visibility,
                        uint8_t *fully_behind, void *workspace, size_t workspace_bytes, void *stream);

/* Feature painting (simulator.py:249-289) straight into
 * the channel-last table: grid (cam, level) has spatial_shape (H, W) =
 * (ceil(img_h / stride), ceil(img_w / stride)) (simulator.py:252-253) and
 * starts at scale_start_index.  entities [n_objects + n_occluders, 9] f64
 * (x, y, z, w, l, h, yaw, cos(yaw), sin(yaw), the trig from the host libm as
 * for msda_visibility): moving objects (signatures [n_objects, C] f64)
 * then occluders (paint nothing).  A cell takes the signature of the nearest
 * entity whose projected rect (visibility.py:46-65) covers its centre.
 * background [rows, C] f64 (the reference's numpy draw: bit-identical
 * output) or NULL (device Philox N(0, sigma) keyed by seed/frame).
 * out [rows, C] of out_dtype = f32(background + signature) (then rounded to
 * f16/bf16).  strides [L] f64, device; spatial_shape_host = host copy.      */
size_t msda_paint_workspace_size(int32_t n_cams, int32_t n_entities);
int32_t msda_paint(const msda_cameras_t *cams, int32_t n_cams, int32_t n_levels, const double *strides,
                   const int32_t *spatial_shape, const int32_t *spatial_shape_host,
                   const int64_t *scale_start_index, int32_t channels, const double *entities,
                   int32_t n_objects, int32_t n_occluders, const double *signatures,
                   const double *background, float sigma, uint64_t seed, int32_t frame, int32_t out_dtype,
                   void *out, void *workspace, size_t workspace_bytes, void *stream);

/* Tracker association cost (tracker.py:105-142), f64,
 * bit-identical to the reference's numpy: geo = |c_q - c_d|, emb = |m_q -
 * e_d| (np.linalg.norm: numpy pairwise summation order), admissible = geo <=
 * gate_radius, cost = alpha_emb*emb + alpha_geo*geo/gate (gate = 1 when
 * gate_radius is infinite), solver_cost = admissible ? cost : 1e9.  Centres
 * [n, 3], embeddings [n, dim] (dim <= 1024), outputs [n_q, n_d], device.   */
int32_t msda_assoc_cost(const double *q_centers, const double *d_centers, const double *q_embeddings,
                        const double *d_embeddings, int32_t n_q, int32_t n_d, int32_t dim, double gate_radius,
                        double alpha_emb, double alpha_geo, double *cost, double *solver_cost,
                        uint8_t *admissible, void *stream);

/* Data-dependent status of the last call that used `workspace` (synchronises
 * `stream`).  detail = the smallest offending query / sample index reported
 * for the winning status code (the reference names the first), or -1.      */
int32_t msda_read_status(const void *workspace, void *stream, int32_t *status, int64_t *detail);

/* ---- host-buffer entry point (end-to-end, copies inside the call) ---- */
typedef struct msda_context msda_context_t;
int32_t msda_context_create(int32_t device, msda_context_t **ctx);
void msda_context_destroy(msda_context_t *ctx);
/* level_data[t] (HOST) points at grid t = cam*n_levels + level, (H, W, C)
 * row-major of `dtype`; spatial_shape (HOST) [n_cams*n_levels*2]; the plan
 * arrays and out / empty are HOST pointers.  Pinned host memory gives
 * asynchronous full-bandwidth copies; pageable memory works but is staged.  */
int32_t msda_csr_host(msda_context_t *ctx, const void *const *level_data, const int32_t *spatial_shape,
                      int32_t n_cams, int32_t n_levels, int32_t channels, int32_t dtype,
                      int64_t n_queries, const int64_t *offsets, const int32_t *camera_index,
                      const int32_t *level, const float *u, const float *v, const float *weight,
                      int32_t precision, int32_t normalize, float *out, uint8_t *empty);

/* bilinear_sample (features.py:184-219) over HOST buffers, on the device:
 * grid (H, W, C) f32 row-major, n cell coordinates u, v (finite; the caller
 * raises for non-finite ones as the reference does), out [n, C] f32 =
 * (c00*w00 + c10*w10) + (c01*w01 + c11*w11) with out-of-grid neighbours
 * reading zero — bit-identical to the reference.  A page-locked grid is read
 * in place; a pageable one is copied.  Synchronous.                         */
int32_t msda_bilinear_host(msda_context_t *ctx, const float *grid, int32_t H, int32_t W, int32_t C, int64_t n,
                           const float *u, const float *v, float *out);

/* Host->device bytes the last msda_csr_host call moved: whole grids copied
 * plus, for large sparsely sampled grids in pinned (device-visible) host
 * memory, only the corner rows the plan touches (fetched over PCIe by the
 * device, once each).                                                       */
long long msda_context_last_h2d_bytes(const msda_context_t *ctx);

/* Offending query (zero weight sum, malformed CSR offsets) or sample (unknown
 * target, non-finite value) of the last msda_csr_host call's non-OK status:
 * the smallest such index, as the reference's sequential loop reports the
 * first (features.py:264-269); -1 when none.                                */
long long msda_context_last_detail(const msda_context_t *ctx);

#ifdef __cplusplus
}
#endif
#endif /* MSDA_B200_H_ */
