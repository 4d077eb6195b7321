/* radsplat.h -- C ABI of the B200-native RadSplat render-and-prune hot path.
 *
 * The reference (fieldsplat, pure NumPy) has no FFI: its boundary is the
 * Python API re-exported at pkg/src/fieldsplat/__init__.py:39-65. Each entry
 * point below replaces one piece of that API's compute; the Python package
 * paper_2403_13806_b200 re-implements the reference signatures on top of it.
 *
 *   rs_render(_ex)       <- render.py:225-287 `_forward` as used by
 *                           rasterize (render.py:290-293),
 *                           rasterize_with_contributions (render.py:296-308;
 *                           max-merge render.py:84-88) and
 *                           rasterize_filtered (render.py:311-315, :241-244)
 *   rs_project           <- render.py:95-158 `_project_arrays`
 *   rs_bin               <- render.py:218-222 `_composite_order` (re-expressed
 *                           as per-tile (depth, index) lists)
 *   rs_blend(_ex)        <- render.py:246-283 compositing loop
 *   rs_compact /
 *   rs_compact_bits      <- np.nonzero of visibility.py:204 indicators /
 *                           io.py:198-243 LSB-first RVIS bitsets
 *   rs_check_finite      <- core.py:522-525 GaussianScene.is_finite
 *   rs_max_merge         <- render.py:84-85 ContributionAccumulator.update
 *   rs_backward          <- render.py:328-487 rasterize_backward +
 *                           _chain_to_parameters (after a training forward)
 *   rs_rspl_unpack /
 *   rs_rspl_pack         <- io.py:128-191 load_scene / save_scene payload
 *                           (RSPL file bytes straight to / from HBM)
 *   rs_pack_bits         <- io.py:198-215 np.packbits(bitorder="little") of
 *                           save_visibility
 *   rs_nearest_cluster   <- visibility.py:80-83 ClusterVisibility.nearest_cluster,
 *                           batched over a trajectory
 *   rs_sq_diff_sum       <- metrics.py:34-45 mse / psnr
 *   rs_ssim              <- metrics.py:59-117 ssim / ssim_with_grad
 *
 * Conventions
 *   - All data pointers are DEVICE pointers (rs_outputs' 64-bit images may be
 *     mapped pinned host memory) owned by the caller; the library
 *     never allocates or frees caller memory. Scratch lives in a caller-provided
 *     workspace sized by rs_workspace_size().
 *   - Every call is stream-ordered on `stream` (a cudaStream_t passed as void*,
 *     NULL = legacy default stream) and never synchronizes the host, so a frame
 *     (rs_render) can be captured into a CUDA graph.
 *   - Re-entrant per workspace; no global mutable state.
 *   - Return value: RS_OK or an RS_E* code (mapped to the reference exception
 *     classes in paper_2403_13806_b200/_native.py).
 *   - Two arithmetic precisions, chosen per frame by rs_options.precision:
 *       RS_F32: fp32 with the operation order of the Tier-A contract
 *               (oracle/cpu_ref.cpp, float tier) -- the fast path;
 *       RS_F64: fp64 with the reference's own expressions and operation order
 *               (render.py:95-158, :250-281) and a contract exp -- results are
 *               bit-identical to the oracle's fp64 contract tier, which matches
 *               the NumPy reference to ~1e-15 (the composite order is the
 *               reference's exact (fp64 depth, index) order).
 *     Cameras and options always cross the boundary in fp64 (the reference's
 *     values); the fp32 path rounds them once (round to nearest).
 */
#ifndef RADSPLAT_H
#define RADSPLAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 2

#if defined(__GNUC__)
#define RS_API __attribute__((visibility("default")))
#else
#define RS_API
#endif

enum {
  RS_OK = 0,
  RS_EINVAL = 1,            /* bad argument (InvalidParameterError)              */
  RS_ENONFINITE = 2,        /* non-finite scene (InvalidSceneError)              */
  RS_ENOMEM_WORKSPACE = 3,  /* workspace too small for n / width / height        */
  RS_ECUDA = 4,             /* CUDA launch error                                 */
  RS_EOVERFLOW = 5          /* more tile pairs than the workspace's pair capacity */
};

/* Storage / arithmetic types (rs_scene.dtype, rs_options.precision). */
enum { RS_F32 = 0, RS_F64 = 1 };

/* Scene in device memory (236 B per Gaussian as fp32, 472 B as fp64):
 *   planes: 11 planes of `plane_stride` values (coalesced per-plane loads)
 *     planes 0-2  positions x,y,z          (core.py:478)
 *     plane  3    opacity logit            (core.py:479; opacity = sigmoid)
 *     planes 4-6  log scales x,y,z         (core.py:481; scale = exp)
 *     planes 7-10 quaternion w,x,y,z       (core.py:482; normalized on device)
 *   sh: n rows of 48 floats, [c][b] at 16*c + b (core.py:480, channel-major
 *     (N,3,16)); each row is read with 128-bit loads, only for visible
 *     Gaussians of frames that produce colour. 16-byte aligned.
 */
typedef struct rs_scene {
  const void* planes; /* float or double (dtype) */
  const void* sh;     /* float or double (dtype) */
  int64_t n;
  int64_t plane_stride;
  int32_t sh_degree; /* 0..3 */
  int32_t dtype;     /* RS_F32 or RS_F64: storage type of planes and sh. Values
                        are widened exactly; an fp64 scene in an RS_F32 frame is
                        rounded to fp32 on load (= numpy astype(float32)). */
} rs_scene;

/* Pinhole camera (core.py:316-374): p_cam = R p + t, row-major R. `center`
 * = -R^T t (core.py:351-354), computed by the caller in fp64. */
typedef struct rs_camera {
  int32_t width, height;
  double fx, fy, cx, cy;
  double R[9];
  double t[3];
  double center[3];
} rs_camera;

/* RasterizeOptions (render.py:37-46) + the arithmetic precision of the frame. */
typedef struct rs_options {
  double alpha_max, alpha_cut, tau_stop, near_limit, lowpass, sigma_bound;
  int32_t precision; /* RS_F32 (fast fp32 contract) or RS_F64 (reference fp64) */
  int32_t _pad;
} rs_options;

/* Image outputs of a colour frame (rs_render_ex / rs_blend_ex). Every pointer
 * may be NULL (that output is skipped); rgb, alpha and count go together.
 *   rgb (H*W*3), alpha, depth (H*W) and count (H*W) int32: device images, fp32
 *     (float*) in RS_F32 frames, fp64 (double*, same fields) in RS_F64 frames.
 *   rgb64 (H*W*3), alpha64 (H*W) float64 and count64 (H*W) int64: the
 *     reference's RenderOutput types (render.py:62-68, :236-239, :283); any
 *     device-dereferenceable memory, typically mapped pinned HOST memory
 *     (cudaHostAlloc; same pointer under UVA) so the blend writes the result
 *     straight over the host link while other tiles are still compositing. */
typedef struct rs_outputs {
  void* rgb;   /* float (RS_F32) or double (RS_F64) */
  void* alpha; /* float or double */
  void* depth; /* float or double */
  int32_t* count;
  double* rgb64;
  double* alpha64;
  int64_t* count64;
  /* training forward (rasterize_cached, render.py:318-321): per pixel the
   * final transmittance and the pair index of its last composited entry
   * (-1: none), which rs_backward walks back from. */
  float* tau;
  int32_t* last;
} rs_outputs;

/* Per-frame counters (device side; copied out by rs_read_stats). */
typedef struct rs_stats {
  uint32_t n_items;     /* Gaussians projected (N, or M for a filtered render) */
  uint32_t n_visible;   /* valid after near / bbox culling                     */
  uint32_t n_pairs;     /* Gaussian-tile overlaps used (min(P, capacity))      */
  uint32_t overflow;    /* 1 if P exceeded the pair capacity: re-run bigger     */
  uint64_t evals;       /* E: bbox-gated evaluations with tau >= tau_stop (only
                           counted when RS_FLAG_COUNT_EVALS is set)            */
  uint64_t composites;  /* C: composited (pixel, Gaussian) pairs (same flag)   */
  uint64_t pairs_needed;/* P, the pair capacity this frame needs               */
  uint32_t bad_index;   /* 1 if active_idx held an index outside [0, n): those
                           entries were skipped; the caller reports RS_EINVAL
                           (InvalidParameterError, render.py:231-234)          */
  uint32_t _pad;
} rs_stats;

/* Device pointers into a workspace, for inspection / parity tests. */
typedef struct rs_buffers {
  const void* records;          /* n_cap x 64 B projected records, item order:
                                   {mx,my,na,nb},{nc,opacity,cut2,depth},
                                   {r,g,b,gid},{x0,x1,y0,y1}                  */
  const void* records64;        /* n_cap x 96 B fp64 records (RS_F64 frames):
                                   mx,my,inv_a,2*inv_b,inv_c,opacity,depth,
                                   ln(alpha_cut/opacity)-1e-6, r,g,b (double),
                                   gid, pad (uint32)                           */
  const uint32_t* items_sorted; /* n_items item ids in (depth, index) order   */
  const uint32_t* pair_items;   /* n_pairs item ids, grouped by tile           */
  const uint32_t* ranges;       /* tiles x 2 : [start, end) into pair_items    */
  const uint32_t* counters;     /* device counters (first words = rs_stats)    */
  int32_t tiles_x, tiles_y;
} rs_buffers;

/* Opaque host-side handle over a caller-allocated device workspace. */
typedef struct rs_workspace rs_workspace;

#define RS_FLAG_COUNT_EVALS 1u /* count E and C (slower; for roofline accounting) */
#define RS_FLAG_BLEND_1PX 2u   /* one pixel per thread blend variant (A/B measurement) */

RS_API int32_t rs_abi_version(void);
RS_API const char* rs_status_string(int32_t status);

/* Bytes of device workspace for scenes of <= n_cap items, <= pair_cap tile
 * pairs and images of <= width x height (tiles_x * tiles_y <= 65536). */
RS_API size_t rs_workspace_size(int64_t n_cap, int64_t pair_cap, int32_t width, int32_t height);

/* Bind a handle to `device_mem` (>= rs_workspace_size bytes, 256-B aligned,
 * owned by the caller). The handle itself is freed by rs_workspace_destroy. */
RS_API int32_t rs_workspace_create(void* device_mem, size_t bytes, int64_t n_cap, int64_t pair_cap, int32_t width,
                            int32_t height, rs_workspace** out);
RS_API void rs_workspace_destroy(rs_workspace* ws);

/* One full frame: project -> depth sort -> tile binning -> blend.
 *   cam:        HOST pointer, uploaded with rs_set_camera; NULL reuses the camera
 *               of the last rs_set_camera -- capture rs_render(cam = NULL) into a
 *               CUDA graph and call rs_set_camera before each replay.
 *   active_idx: optional ascending list of m scene indices (filtered render:
 *               only listed Gaussians are projected); NULL = all scene->n.
 *   out_rgb (H*W*3), out_alpha, out_depth (H*W), out_count (H*W int32): may
 *               all be NULL for a score-only (importance) pass.
 *               Out-of-range entries are skipped and flagged (rs_stats.bad_index).
 *   out_rgb (H*W*3), out_alpha, out_depth (H*W), out_count (H*W int32): may
 *               all be NULL for a score-only (importance) pass; float images in
 *               RS_F32 frames, double in RS_F64 frames.
 *   scores:     optional n values max-merged with each Gaussian's max alpha*tau
 *               (render.py:273-275): uint32 bit patterns of non-negative floats
 *               (RS_F32) or uint64 bit patterns of non-negative doubles (RS_F64).
 */
RS_API int32_t rs_render(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m, const rs_camera* cam,
                  const rs_options* opts, void* out_rgb, void* out_alpha, void* out_depth, int32_t* out_count,
                  void* scores, uint32_t flags, void* stream);

/* rs_render with the image outputs of an rs_outputs (NULL = score-only frame). */
RS_API int32_t rs_render_ex(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                            const rs_camera* cam, const rs_options* opts, const rs_outputs* out, void* scores,
                            uint32_t flags, void* stream);

/* Stream-ordered camera upload into the workspace (also fixes the image size of
 * the following frames); `cam` may be reused as soon as the call returns. */
RS_API int32_t rs_set_camera(rs_workspace* ws, const rs_camera* cam, void* stream);

/* Stages of rs_render, callable separately (same workspace state machine). */
RS_API int32_t rs_project(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m, const rs_camera* cam,
                   const rs_options* opts, void* stream);
RS_API int32_t rs_bin(rs_workspace* ws, void* stream);
/* rs_project that also writes, per item (culled included), the reference's
 * ProjectedGaussian fields (render.py:49-59) as 16 values (float in RS_F32,
 * double in RS_F64 frames) {mx, my, a, b, c, inv_a, inv_b, inv_c, radius,
 * depth, r, g, b, opacity, valid, cut} to out_proj and {x0, x1, y0, y1} to
 * out_bbox (render.py:161-211). */
RS_API int32_t rs_project_full(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                        const rs_camera* cam, const rs_options* opts, void* out_proj, int32_t* out_bbox,
                        void* stream);
/* rs_blend / rs_blend_ex: `opts` must have the precision of the rs_project call. */
RS_API int32_t rs_blend(rs_workspace* ws, const rs_options* opts, void* out_rgb, void* out_alpha, void* out_depth,
                 int32_t* out_count, void* scores, uint32_t flags, void* stream);
RS_API int32_t rs_blend_ex(rs_workspace* ws, const rs_options* opts, const rs_outputs* out, void* scores,
                           uint32_t flags, void* stream);

/* Gradients of a scalar loss through the image of the frame the last
 * rs_render_ex on this workspace produced with rs_outputs tau / last (the
 * training forward, render.py:318-321): grad_image = dL/dcolor (H*W*3, device),
 * outputs per scene Gaussian (device, zeroed here): positions (n,3), sh (n,48),
 * log-scales (n,3), quaternions (n,4), opacity logits (n), |dL/dmean2d| (n),
 * touched (n bytes). Same scene / active list as that forward. RS_F32 frames
 * of fp32 scenes only (RS_EINVAL otherwise); the per-Gaussian sums are
 * atomics, so results match the reference to a tolerance, not bit for bit. */
RS_API int32_t rs_backward(rs_workspace* ws, const rs_scene* scene, const int32_t* active_idx, int64_t m,
                           const rs_options* opts, const float* grad_image, const float* tau, const int32_t* last,
                           float* g_pos, float* g_sh, float* g_ls, float* g_quat, float* g_logit, float* g_mean2d,
                           uint8_t* touched, void* stream);

/* Copy the device counters to host memory (synchronizes `stream`). */
RS_API int32_t rs_read_stats(rs_workspace* ws, rs_stats* out, void* stream);
/* Did any frame since the last reset overflow its pair capacity, and the
 * largest P such a frame needed (synchronizes `stream`; reset != 0 clears
 * the record). Lets a batch of frames -- a scoring pass -- run without a
 * host sync per frame and be checked once. rs_read_sticky also reports
 * whether any of those frames skipped an out-of-range active_idx entry. */
RS_API int32_t rs_read_overflow(rs_workspace* ws, uint32_t* out_overflowed, uint64_t* out_pairs_needed_max,
                                int32_t reset, void* stream);
RS_API int32_t rs_read_sticky(rs_workspace* ws, uint32_t* out_overflowed, uint64_t* out_pairs_needed_max,
                              uint32_t* out_bad_index, int32_t reset, void* stream);
RS_API int32_t rs_get_buffers(rs_workspace* ws, rs_buffers* out);

/* Stable compaction: indices i (ascending) with flags[i] != 0, count -> *out_count (device). */
RS_API size_t rs_compact_workspace_size(int64_t n);
RS_API int32_t rs_compact(const uint8_t* flags, int64_t n, int32_t* out_idx, uint32_t* out_count, void* scratch,
                   size_t scratch_bytes, void* stream);
/* Same from an LSB-first bitset (bit i of byte i/8; io.py:205-206). */
RS_API int32_t rs_compact_bits(const uint8_t* bits, int64_t n, int32_t* out_idx, uint32_t* out_count, void* scratch,
                        size_t scratch_bytes, void* stream);

/* *out_bad (device) = number of non-finite scene values (planes and SH rows,
 * either dtype; 0 = finite). */
RS_API int32_t rs_check_finite(const rs_scene* scene, uint32_t* out_bad, void* stream);

/* RSPL payload (device, 16-B aligned: positions (n,3), log-scales (n,3),
 * quaternions w-x-y-z (n,4), opacity logits (n), SH (n,48), fp32) -> device
 * scene planes (see rs_scene) + SH rows; quaternions normalized in fp64 like
 * the reference's GaussianScene (core.py:111-117), *out_bad (device) = number
 * of zero quaternions. rs_rspl_pack is the inverse. */
RS_API int32_t rs_rspl_unpack(const float* payload, int64_t n, float* planes, int64_t plane_stride, float* sh,
                              uint32_t* out_bad, void* stream);
RS_API int32_t rs_rspl_pack(const float* planes, int64_t plane_stride, const float* sh, int64_t n, float* payload,
                            void* stream);
/* n flags (bytes, nonzero = set) -> ceil(n/8) bytes of LSB-first bits (RVIS indicator). */
RS_API int32_t rs_pack_bits(const uint8_t* flags, int64_t n, uint8_t* bits, void* stream);

/* out[i] = index of the centre (k x 3, float64) nearest to position i (m x 3,
 * float64): Euclidean distance as np.linalg.norm, lowest index on ties. */
RS_API int32_t rs_nearest_cluster(const double* centers, int32_t k, const double* positions, int64_t m, int32_t* out,
                                  void* stream);

/* sum of (a - b)^2 over n float64 values (device) -> *out_sum (device). */
RS_API int32_t rs_sq_diff_sum(const double* a, const double* b, int64_t n, double* out_sum, void* stream);
/* SSIM of (H, W, C) float64 images x, y (device, channels last): *out_sum = the
 * sum of the per-window SSIM over all 'valid' windows and channels (divide by
 * (H-win+1)(W-win+1)C for the reference's mean); `kernel` = the win x win
 * Gaussian window (device, float64, metrics.py:48-52). With `grad` (H*W*C,
 * device) also dSSIM/dx; that needs a scratch of rs_ssim_workspace_size bytes. */
RS_API size_t rs_ssim_workspace_size(int32_t height, int32_t width, int32_t channels, int32_t win);
RS_API int32_t rs_ssim(const double* x, const double* y, int32_t height, int32_t width, int32_t channels,
                       int32_t win, const double* kernel, double* out_sum, double* grad, void* scratch,
                       size_t scratch_bytes, void* stream);

/* dst[i] = max(dst[i], src[i]) over n non-negative floats. */
RS_API int32_t rs_max_merge(float* dst, const float* src, int64_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RADSPLAT_H */
