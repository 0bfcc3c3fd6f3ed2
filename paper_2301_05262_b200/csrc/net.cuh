// Plan layer: the device-resident, kernel-layout form of a NetworkConfig +
// weight dict (network.py:44-144, 277-285).
#pragma once

#include <string>
#include <vector>

#include "common.cuh"

namespace nsm {

constexpr int kMaxLevels = 8;

struct ConvW {
    int cin = 0, cout = 0, k = 0;
    const float* w32 = nullptr;   // OIHW fp32 (reference layout)
    const float* b32 = nullptr;   // (O,) fp32
    const void* wpk = nullptr;    // packed 16-bit tiles for the tensor-core path
    bool present() const { return k != 0; }
};

struct Level {
    ConvW enc3, enc1, dec3, dec1;
};

struct Plan {
    nsm_net_config cfg{};
    nsm_dtype act = NSM_F32;
    int nlev = 0;                 // len(level_channels)
    int chans[kMaxLevels] = {};
    int first_in = 0;
    int out_ch = 0;
    Level lev[kMaxLevels];
    ConvW head;
    // level-0 decoder in polyphase form on the level-1 grid (dec0p_kernel):
    // conv3(up2(x)) = 4 phase convolutions of x, stacked along N (4 x 16);
    // dec1 and the head as phase-block-diagonal 1x1 convs (K = 64)
    ConvW d0p3, d0p1, d0ph;
    int64_t n_params = 0;
    void* dev = nullptr;          // one allocation holding every tensor
    int device = -1;              // the CUDA device dev lives on
    size_t dev_bytes = 0;
};

size_t forward_f32_workspace(const Plan& p, int n, int h, int w);
nsm_status forward_f32(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws,
                       size_t ws_bytes, cudaStream_t st);

// generic fp16 / bf16 tensor-core path for any NetworkConfig (net_gen16.cu)
size_t forward_gen16_workspace(const Plan& p, int n, int h, int w);
nsm_status forward_gen16(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws,
                         size_t ws_bytes, cudaStream_t st);

// fp16 / bf16 tensor-core path (net_f16.cu)
bool f16_supported(const Plan& p);
size_t infer_f16_workspace(const Plan& p, int n, int h, int w);
nsm_status pack_f16(Plan& p, std::vector<char>& host_blob, size_t& offset_out);
nsm_status forward_f16(const Plan& p, const float* x, int n, int h, int w, float* out, void* ws,
                       size_t ws_bytes, cudaStream_t st);
nsm_status infer_f16(const Plan& p, const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                     const nsm_frame* frames, int n, int h, int w, void* y, nsm_dtype y_dtype,
                     int64_t* first_bad, int32_t* texel_idx, void* ws, size_t ws_bytes, cudaStream_t st);

nsm_status launch_features(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                           const nsm_frame* frames, int32_t n, int32_t h, int32_t w, int32_t ho,
                           int32_t wo, float* out, int32_t* tidx, int64_t* first_bad,
                           cudaStream_t st);
void launch_fill_i64(int64_t* p, int n, int64_t v, cudaStream_t st);
// feat5.cu: the 4 planes + the blocker-search penumbra plane.  out_kind 0/1:
// fp16 / bf16 chunk-planar level-0 tensor (nf, 3, H0, W0, 8); 2: fp32 planes
// (nf, 5, h, w).  first_bad pre-filled by the caller.
nsm_status launch_feat5(const nsm_gbuffer* g, const float* sm, int64_t sm_stride, const nsm_frame* frames,
                        int nf, int h, int w, int H0, int W0, void* out, int out_kind, int64_t* first_bad,
                        int32_t* tidx, cudaStream_t st, int32_t* dbg = nullptr);
nsm_status launch_blocker(const nsm_gbuffer* g, const float* sm, int64_t sm_stride, const nsm_frame* frames,
                          int32_t n, int32_t h, int32_t w, int32_t radius, float* out, int64_t* first_bad,
                          cudaStream_t st);
nsm_status launch_motion(const nsm_gbuffer* g, const nsm_camera* cams, int t_frames, int h, int w,
                         double* vec, uint8_t* valid, cudaStream_t st);
nsm_status launch_instability(const float* vis, const double* vec, const uint8_t* valid, int t_frames,
                              int h, int w, double alpha, double* acc, unsigned long long* cnt,
                              cudaStream_t st);
nsm_status launch_render_gbuffer(const double* prims, int32_t n_prims, const nsm_camera* cam,
                                 float* d, float* normal, float* position, cudaStream_t st);
nsm_status launch_render_shadowmap(const double* prims, int32_t n_prims,
                                   const nsm_emitter_view* view, float* depth, cudaStream_t st);

}  // namespace nsm
