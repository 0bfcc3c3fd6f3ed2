/*
 * nsm.h -- C ABI of the B200 (sm_100a) neural-shadow-mapping inference path.
 *
 * The path is the per-frame inference of the reference package `shadowkit`
 * (/root/reference/pkg/src/shadowkit): stage 1 `raster.assemble_features`
 * (G-buffer + shadow map -> 4 input planes) and stage 2 `network.forward`
 * (compact space-to-depth U-Net -> visibility in [0, 1]).  Every entry point
 * below replaces one reference interface; the file:line it replaces is given
 * beside it.  No torch / C++ types cross this boundary: plain pointers, sizes
 * and POD structs.  Device pointers are caller-owned (e.g. torch CUDA tensors);
 * the library never allocates per call (the plan owns its packed weights).
 *
 * Errors: every call returns an nsm_status; `nsm_last_error()` gives the
 * thread-local message.  The Python host maps the codes back onto the
 * reference's exception types:
 *   NSM_ERR_SHAPE   -> ValueError    (network.py:169-173 messages)
 *   NSM_ERR_FRUSTUM -> raster.FrustumError (raster.py:60-61, 251-255)
 *   NSM_ERR_FORMAT  -> fileio.FormatError  (fileio.py:22-23, network.py:272-273)
 *   NSM_ERR_ARG     -> ValueError
 *   NSM_ERR_CUDA    -> RuntimeError
 * Thread safety: a plan is immutable after nsm_plan_create and may be used
 * from several host threads on distinct streams with distinct workspaces.
 */
#ifndef NSM_H
#define NSM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSM_ABI_VERSION 2
#define NSM_MAX_FRAMES_PER_LAUNCH 8

typedef enum nsm_status {
    NSM_OK = 0,
    NSM_ERR_ARG = 1,
    NSM_ERR_SHAPE = 2,
    NSM_ERR_FRUSTUM = 3,
    NSM_ERR_FORMAT = 4,
    NSM_ERR_CUDA = 5,
    NSM_ERR_UNSUPPORTED = 6
} nsm_status;

typedef enum nsm_dtype {
    NSM_F32 = 0,   /* reference precision (fp32 oracle parity, <= 1e-4)   */
    NSM_F16 = 1,   /* fp16 operands, fp32 accumulate (<= 1e-2 / 1e-4 MSE) */
    NSM_BF16 = 2,  /* bf16 operands, fp32 accumulate                      */
    NSM_F64 = 3    /* G-buffer planes only (drop-in of fp64 numpy buffers) */
} nsm_dtype;

/* network.NetworkConfig (network.py:44-76). */
typedef struct nsm_net_config {
    int32_t layers;
    int32_t base_channels;
    int32_t in_channels;
    int32_t use_space_to_depth;
    int32_t channel_cap;
} nsm_net_config;

/* raster.EmitterView (raster.py:64-73): square frustum from the emitter
 * centre; `height`/`width` is the shadow-map resolution. */
typedef struct nsm_emitter_view {
    double position[3];
    double forward[3];
    double up[3];
    double right[3];
    double tan_half;
    int32_t height;
    int32_t width;
} nsm_emitter_view;

/* scene.CameraPose (scene.py:102-114); forward/up already orthonormal. */
typedef struct nsm_camera {
    double position[3];
    double forward[3];
    double up[3];
    double fov_y;
    int32_t height;
    int32_t width;
} nsm_camera;

/* Per-frame constants of one frame in a batch. */
typedef struct nsm_frame {
    nsm_camera camera;
    nsm_emitter_view view;
    double emitter_center[3];
    double size_index;   /* ch2 dc offset (raster.py:276), no range check */
    double bias;         /* acne bias b; ShadowMap.default_bias = 1e-3 * diag */
} nsm_frame;

/* raster.GBuffer (raster.py:154-170) as planar device buffers of one batch:
 * frame f, plane element (y, x) of d is d[f * frame_stride + y * W + x];
 * normal / position are (3, H, W) per frame at the same frame_stride * 3.
 * z_f / c_e / c_c / coverage are optional: when NULL they are derived from
 * the planes exactly as render_gbuffer does (raster.py:222-232) and coverage
 * is d > 0. */
typedef struct nsm_gbuffer {
    nsm_dtype dtype;            /* NSM_F32 or NSM_F64 */
    const void* d;
    const void* normal;
    const void* position;
    const void* z_f;
    const void* c_e;
    const void* c_c;
    const uint8_t* coverage;
    int64_t frame_stride;       /* elements per (H, W) plane-set of one frame */
} nsm_gbuffer;

typedef struct nsm_plan nsm_plan;

/* ---- plan layer: network.init_weights / load_network -> kernel layout ----
 * Replaces the weight dict consumed by network.forward (network.py:165-195;
 * names/shapes per network._named_params, network.py:277-285).  host_data[i]
 * is an fp32 OIHW (weights) or (O,) (bias) array of shape dims[i][0..ndims[i]).
 * A name set or shape that does not match cfg -> NSM_ERR_FORMAT
 * (network.py:271-273); an invalid cfg -> NSM_ERR_ARG (network.py:52-58). */
nsm_status nsm_plan_create(const nsm_net_config* cfg, int32_t n_tensors,
                           const char* const* names, const float* const* host_data,
                           const int32_t* ndims, const int32_t* const* dims,
                           nsm_dtype act_dtype, nsm_plan** out_plan);
void nsm_plan_destroy(nsm_plan* plan);
nsm_status nsm_plan_info(const nsm_plan* plan, nsm_net_config* cfg, nsm_dtype* act_dtype,
                         int64_t* n_params);

/* Device workspace needed by nsm_forward / nsm_infer for a batch of n frames
 * of h x w input pixels. */
size_t nsm_workspace_size(const nsm_plan* plan, int32_t n, int32_t h, int32_t w);

/* ---- stage 1: raster.assemble_features (raster.py:266-278) ----
 * out_planes: (n, 4, h, w) fp32 device.  texel_idx (nullable): (n, 2, h, w)
 * int32 (row, col) nearest texels, -1 on uncovered pixels.  first_bad: n
 * device int64 = row-major index of the first covered pixel that projects
 * outside the frustum, INT64_MAX if none (raster.py:251-255); the call
 * itself does not synchronise, the host raises FrustumError after reading it.
 * sm: (n, Hs, Ws) fp32 radial depths, +inf = miss, frame f at f * sm_stride. */
nsm_status nsm_features(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                        const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                        float* out_planes, int32_t* texel_idx, int64_t* first_bad,
                        void* stream);

/* ---- blocker-search penumbra plane (BASELINE configs 3/4 extension) ----
 * No reference implementation (PCSS is out of the reference's scope,
 * SPEC.md:14): per covered pixel the nearest texel of _shadow_lookup, a
 * (2*radius)^2 texel window, blockers = finite depths < z_f - bias,
 * (z_min, z_max) -> analysis.penumbra_extents (analysis.py:240-269) with
 * r_e = size_index * 0.0625 m, width (x_a + x_b) * focal_px / d
 * (analysis.py:319-320) in units of the focal length: (x_a + x_b) / d
 * (resolution independent).  out: (n, h, w) fp32, the 5th input plane of a
 * NetworkConfig(in_channels=5) net.  first_bad as nsm_features. */
nsm_status nsm_blocker_plane(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                             const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                             int32_t radius, float* out, int64_t* first_bad, void* stream);

/* ---- stage 1 of the 5-plane net: the 4 planes + the blocker plane ----
 * The feature pass of NetworkConfig(in_channels=5) plans (BASELINE configs
 * 3/4 "soft shadows"): the 4 planes of assemble_features plus the blocker-
 * search penumbra plane (definition as nsm_blocker_plane, radius 8: a 16 x 16
 * texel window), in one pass with the map windows staged in shared memory.
 * out_planes: (n, 5, h, w) fp32 device.  Planes 0-3 use the fused hot path's
 * fp32 arithmetic (nsm_features is the fp64-faithful 4-plane drop-in);
 * texel_idx / first_bad as nsm_infer_ex / nsm_features. */
nsm_status nsm_features5(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                         const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                         float* out_planes, int32_t* texel_idx, int64_t* first_bad, void* stream);

/* ---- stage 2: network.forward (network.py:165-209) ----
 * x: (n, in_channels, h, w) fp32 device, y: (n, 1, h, w) fp32 device.
 * h, w must be divisible by 2**(layers-1) (NSM_ERR_SHAPE otherwise). */
nsm_status nsm_forward(const nsm_plan* plan, const float* x, int32_t n, int32_t h,
                       int32_t w, float* y, void* workspace, size_t ws_bytes, void* stream);

/* ---- fused stages 1+2: the hot path ----
 * assemble_features then forward per frame, features never written to HBM
 * on the fp16/bf16 plans of 4-plane nets.  A NetworkConfig(in_channels=5)
 * plan (16-bit only) adds the blocker-search plane (nsm_features5); its
 * feature pass writes a 16-bit s2d tensor that the level-0 encoder reads.  h need not be divisible by 2**(layers-1): rows /
 * columns up to the next multiple are treated as uncovered (zero features,
 * the same padding the oracle applies) and cropped from y.  y: (n, 1, h, w)
 * of y_dtype (NSM_F32 or NSM_F16). */
nsm_status nsm_infer(const nsm_plan* plan, const nsm_gbuffer* g, const float* sm,
                     int64_t sm_stride, const nsm_frame* frames, int32_t n, int32_t h,
                     int32_t w, void* y, nsm_dtype y_dtype, int64_t* first_bad,
                     void* workspace, size_t ws_bytes, void* stream);

/* nsm_infer plus the parity hook of the fused feature pass: texel_idx
 * (nullable) is an (n, 2, h, w) int32 device array that receives, for every
 * covered pixel, the (row, col) shadow-map texel the fused kernel actually
 * gathered -- the np.rint indices of _shadow_lookup (raster.py:247-250) --
 * so tests can prove them bit-exact.  Uncovered pixels are either left
 * untouched or set to -1 (the caller pre-fills with -1).  Same validation and errors as
 * nsm_infer; with texel_idx == NULL the two calls are identical. */
nsm_status nsm_infer_ex(const nsm_plan* plan, const nsm_gbuffer* g, const float* sm,
                        int64_t sm_stride, const nsm_frame* frames, int32_t n, int32_t h,
                        int32_t w, void* y, nsm_dtype y_dtype, int64_t* first_bad,
                        int32_t* texel_idx, void* workspace, size_t ws_bytes, void* stream);

/* ---- input producers (the step before the path) ----
 * raster.render_gbuffer (raster.py:217-242) depth/normal/position planes and
 * raster.render_shadowmap (raster.py:206-214) over an analytic primitive
 * table: prims = device (n_prims, 16) fp64 rows, see scenes.primitive_table. */
nsm_status nsm_render_gbuffer(const double* prims, int32_t n_prims, const nsm_camera* cam,
                              float* d, float* normal, float* position, void* stream);
nsm_status nsm_render_shadowmap(const double* prims, int32_t n_prims,
                                const nsm_emitter_view* view, float* depth, void* stream);

/* ---- temporal consumers of the visibility ----
 * nsm_motion_vectors: raster.motion_vectors (raster.py:330-358) for every
 * consecutive pair of a t_frames sequence: pair k = (frame k, frame k+1),
 * frame k+1's points reprojected with cams[k] (camera of frame k).  g holds
 * t_frames frames (frame_stride as above; coverage NULL -> d > 0).
 * vec: (t_frames-1, 2, h, w) fp64 (row, col) offsets, 0 on uncovered pixels;
 * valid: (t_frames-1, h, w) uint8.
 * nsm_temporal_instability: the per-pair sums of
 * analysis.temporal_instability (analysis.py:350-377): vis (t_frames, h, w)
 * fp32, acc (t_frames-1) fp64 sums of expm1(alpha |cur - prev[reproj]|) over
 * valid pixels, count (t_frames-1) uint64 valid pixels.  E = sum(acc) /
 * sum(count); the host raises NoValidPixels when sum(count) == 0. */
nsm_status nsm_motion_vectors(const nsm_gbuffer* g, const nsm_camera* cams, int32_t t_frames,
                              int32_t h, int32_t w, double* vec, uint8_t* valid, void* stream);
nsm_status nsm_temporal_instability(const float* vis, const double* vec, const uint8_t* valid,
                                    int32_t t_frames, int32_t h, int32_t w, double alpha,
                                    double* acc, uint64_t* count, void* stream);

/* ---- tracing / launch accounting (tracing) ----
 * nsm_launch_count: kernels launched by this library since load (graph
 * replays not included).  nsm_profile_enable(1): record a CUDA-event pair
 * on the launching stream around every eager (non-captured) launch;
 * nsm_profile_report writes "name launches total_ms" lines into buf, clears
 * the records and returns the full report length. */
int64_t nsm_launch_count(void);
void nsm_profile_enable(int32_t on);
int32_t nsm_profile_report(char* buf, size_t cap);

const char* nsm_last_error(void);
int32_t nsm_abi_version(void);

/* Build flavour: bit 0 set = experiment build (-DNSM_EXPERIMENTS: the NSM_*
 * attribution switches of tools/, which skip work and give wrong results).
 * Release builds ignore every NSM_* environment variable; bench.py refuses
 * to time an experiment build. */
#define NSM_BUILD_EXPERIMENTS 1
int32_t nsm_build_flags(void);

#ifdef __cplusplus
}
#endif
#endif /* NSM_H */
