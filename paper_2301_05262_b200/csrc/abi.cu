// The extern "C" boundary (include/nsm.h): argument validation, the plan
// layer (network.py:44-144, 267-285 semantics) and dispatch to the kernels.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"
#include "net.cuh"
#include "prof.cuh"

namespace nsm {

namespace {
thread_local std::string g_err;
#ifdef NSM_EXPERIMENTS
int32_t* g_feat5_dbg = nullptr;   // nsm_debug_feat5: per-pixel search record of nsm_features5
#else
constexpr int32_t* g_feat5_dbg = nullptr;
#endif
}

nsm_status fail(nsm_status code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

void clear_error() { g_err.clear(); }

void make_frame_table(const nsm_frame* frames, int32_t n, FrameTable& tab) {
    memset(&tab, 0, sizeof tab);
    for (int i = 0; i < n; ++i) {
        const nsm_frame& s = frames[i];
        FrameK& f = tab.f[i];
        for (int a = 0; a < 3; ++a) {
            f.vp[a] = s.view.position[a];
            f.vf[a] = s.view.forward[a];
            f.vu[a] = s.view.up[a];
            f.vr[a] = s.view.right[a];
            f.cp[a] = s.camera.position[a];
            f.cf[a] = s.camera.forward[a];
            f.cu[a] = s.camera.up[a];
            f.ec[a] = s.emitter_center[a];
        }
        // CameraPose.right = forward x up (scene.py:143-145)
        f.cr[0] = s.camera.forward[1] * s.camera.up[2] - s.camera.forward[2] * s.camera.up[1];
        f.cr[1] = s.camera.forward[2] * s.camera.up[0] - s.camera.forward[0] * s.camera.up[2];
        f.cr[2] = s.camera.forward[0] * s.camera.up[1] - s.camera.forward[1] * s.camera.up[0];
        f.tan_half = s.view.tan_half;
        f.hs = s.view.height;
        f.ws = s.view.width;
        f.half_h = std::tan(s.camera.fov_y / 2.0);
        f.half_w = f.half_h * ((double)s.camera.width / s.camera.height);
        f.ch = s.camera.height;
        f.cw = s.camera.width;
        f.size_index = s.size_index;
        f.bias = s.bias;
        f.pa = s.view.width / (2.0 * s.view.tan_half);
        f.pb = s.view.width / 2.0 - 0.5;
        f.qa = s.view.height / (2.0 * s.view.tan_half);
        f.qb = s.view.height / 2.0 - 0.5;
        for (int a = 0; a < 3; ++a) {
            f.fec[a] = (float)f.ec[a];
            f.fcf[a] = (float)f.cf[a];
            f.fcr[a] = (float)f.cr[a];
            f.fcu[a] = (float)f.cu[a];
        }
        f.fu1 = (float)(2.0 * f.half_w / f.cw);
        f.fu0 = (float)(f.half_w / f.cw - f.half_w);
        f.fw1 = (float)(-2.0 * f.half_h / f.ch);
        f.fw0 = (float)(f.half_h - f.half_h / f.ch);
        f.fbias = (float)f.bias;
        f.fsize = (float)f.size_index;
        // affine forms: pa * (p - vp).vr, -qa * (p - vp).vu, (p - vp).vf
        double cx = 0, cy = 0, cz = 0;
        for (int a = 0; a < 3; ++a) {
            f.kx[a] = f.pa * f.vr[a];
            f.ky[a] = -f.qa * f.vu[a];
            f.kz[a] = f.vf[a];
            cx -= f.vr[a] * f.vp[a];
            cy -= f.vu[a] * f.vp[a];
            cz -= f.vf[a] * f.vp[a];
            f.fcp[a] = (float)f.cp[a];
        }
        f.kx[3] = f.pa * cx;
        f.ky[3] = -f.qa * cy;
        f.kz[3] = cz;
    }
}

namespace {

struct Spec {
    int cout, cin, k;
};

// network._level_plan (network.py:98-118) + _named_params (:277-285).
bool level_plan(const nsm_net_config& c, Plan& p, std::map<std::string, Spec>& names) {
    p.nlev = c.use_space_to_depth ? c.layers - 1 : c.layers;
    if (p.nlev < 1 || p.nlev > kMaxLevels) return false;
    for (int j = 0; j < p.nlev; ++j) {
        long long v = (long long)c.base_channels << j;
        p.chans[j] = (int)std::min<long long>(v, c.channel_cap);
    }
    p.first_in = c.use_space_to_depth ? 4 * c.in_channels : c.in_channels;
    p.out_ch = c.use_space_to_depth ? 4 : 1;
    auto add = [&](int j, const char* tag, ConvW& cw, int cin, int cout, int k) {
        cw.cin = cin;
        cw.cout = cout;
        cw.k = k;
        std::string base = "l" + std::to_string(j) + "." + tag;
        names[base + ".w"] = {cout, cin, k};
        names[base + ".b"] = {cout, -1, 0};
    };
    for (int j = 0; j < p.nlev; ++j) {
        const int cin = j == 0 ? p.first_in : p.chans[j - 1];
        const int cj = p.chans[j];
        if (j == p.nlev - 1) {
            const int cdown = p.nlev > 1 ? p.chans[j - 1] : p.chans[0];
            add(j, "enc3", p.lev[j].enc3, cin, cj, 3);
            add(j, "enc1", p.lev[j].enc1, cj, cdown, 1);
        } else {
            const int cout = j > 0 ? p.chans[j - 1] : p.chans[0];
            add(j, "enc3", p.lev[j].enc3, cin, cj, 3);
            add(j, "enc1", p.lev[j].enc1, cj, cj, 1);
            add(j, "dec3", p.lev[j].dec3, cj, cj, 3);
            add(j, "dec1", p.lev[j].dec1, cj, cout, 1);
        }
    }
    p.head.cin = p.chans[0];
    p.head.cout = p.out_ch;
    p.head.k = 1;
    names["head.w"] = {p.out_ch, p.chans[0], 1};
    names["head.b"] = {p.out_ch, -1, 0};
    return true;
}

ConvW* conv_by_name(Plan& p, const std::string& base) {
    if (base == "head") return &p.head;
    int j;
    char tag[8];
    if (sscanf(base.c_str(), "l%d.%7s", &j, tag) != 2 || j < 0 || j >= p.nlev) return nullptr;
    Level& L = p.lev[j];
    if (!strcmp(tag, "enc3")) return &L.enc3;
    if (!strcmp(tag, "enc1")) return &L.enc1;
    if (!strcmp(tag, "dec3")) return &L.dec3;
    if (!strcmp(tag, "dec1")) return &L.dec1;
    return nullptr;
}

nsm_status check_stream_err() {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(NSM_ERR_CUDA, "CUDA error: %s", cudaGetErrorString(e));
    return NSM_OK;
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

// crop (n, 1, hp, wp) fp32 -> (n, 1, h, w) of the requested dtype
__global__ void crop_kernel(const float* __restrict__ src, int hp, int wp, int h, int w, int n,
                            void* __restrict__ dst, int f16) {
    const int64_t total = (int64_t)n * h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int x = i % w, y = (i / w) % h;
        const int64_t f = i / ((int64_t)h * w);
        const float v = src[(f * hp + y) * wp + x];
        if (f16)
            reinterpret_cast<__half*>(dst)[i] = __float2half_rn(v);
        else
            reinterpret_cast<float*>(dst)[i] = v;
    }
}

// Every frame of a batch must describe the (h, w) frames the planes hold
// and a shadow map that fits its sm_stride slot (the kernels index the map
// with each frame's own resolution; a single frame needs no stride).
nsm_status check_frames(const nsm_frame* frames, int32_t n, int32_t h, int32_t w, int64_t sm_stride) {
    for (int i = 0; i < n; ++i) {
        const nsm_frame& f = frames[i];
        if (f.camera.height != h || f.camera.width != w)
            return fail(NSM_ERR_ARG, "frame %d: camera is %dx%d but the G-buffer planes are %dx%d", i,
                        f.camera.height, f.camera.width, h, w);
        if (f.view.height <= 0 || f.view.width <= 0 || (n > 1 && (int64_t)f.view.height * f.view.width > sm_stride))
            return fail(NSM_ERR_ARG, "frame %d: a %dx%d shadow map does not fit sm_stride %lld", i,
                        f.view.height, f.view.width, (long long)sm_stride);
    }
    return NSM_OK;
}

// A plan's weights live on the device that was current at creation.
nsm_status check_device(const Plan& p) {
    int dev = -1;
    cudaGetDevice(&dev);
    if (dev != p.device)
        return fail(NSM_ERR_ARG, "plan lives on device %d, current device is %d", p.device, dev);
    return NSM_OK;
}

// the unfused path of nsm_infer: fp32 feature planes (padded), the forward's
// workspace, the padded visibility (fp32 plans and the generic 16-bit ones)
size_t forward_any_workspace(const Plan& p, int n, int h, int w) {
    return p.act == NSM_F32 ? forward_f32_workspace(p, n, h, w) : forward_gen16_workspace(p, n, h, w);
}

size_t infer_f32_workspace(const Plan& p, int n, int h, int w) {
    const int m = 1 << (p.cfg.layers - 1);
    const int hp = round_up(h, m), wp = round_up(w, m);
    return (size_t)n * 4 * hp * wp * 4 + (size_t)n * hp * wp * 4 + 256 +
           forward_any_workspace(p, n, hp, wp);
}

}  // namespace
}  // namespace nsm

using namespace nsm;

extern "C" {

int32_t nsm_abi_version(void) { return NSM_ABI_VERSION; }

#ifdef NSM_EXPERIMENTS
// Debug hook of experiment builds (not in nsm.h): the next nsm_features5
// calls also write (zmin, zmax, thr, path) per pixel into buf ((n, h, w, 4)
// int32, device); tools/dbg5.py.
void nsm_debug_feat5(int32_t* buf) { g_feat5_dbg = buf; }
#endif

int32_t nsm_build_flags(void) {
#ifdef NSM_EXPERIMENTS
    return NSM_BUILD_EXPERIMENTS;
#else
    return 0;
#endif
}

const char* nsm_last_error(void) { return g_err.c_str(); }

nsm_status nsm_plan_create(const nsm_net_config* cfg, int32_t n_tensors, const char* const* names,
                           const float* const* host_data, const int32_t* ndims,
                           const int32_t* const* dims, nsm_dtype act_dtype, nsm_plan** out_plan) {
    clear_error();
    if (!cfg || !out_plan || n_tensors < 0 || (n_tensors && (!names || !host_data || !ndims || !dims)))
        return fail(NSM_ERR_ARG, "nsm_plan_create: null argument");
    *out_plan = nullptr;
    // NetworkConfig.__post_init__ (network.py:52-58)
    if (cfg->layers < 2) return fail(NSM_ERR_ARG, "network needs layers >= 2");
    if (cfg->base_channels < 4) return fail(NSM_ERR_ARG, "base_channels must be >= 4");
    if (cfg->in_channels < 1) return fail(NSM_ERR_ARG, "in_channels must be >= 1");
    if (cfg->channel_cap < 1) return fail(NSM_ERR_ARG, "channel_cap must be >= 1");
    if (act_dtype != NSM_F32 && act_dtype != NSM_F16 && act_dtype != NSM_BF16)
        return fail(NSM_ERR_ARG, "act_dtype must be F32, F16 or BF16");
    Plan* p = new Plan();
    p->cfg = *cfg;
    p->act = act_dtype;
    std::map<std::string, Spec> expect;
    if (!level_plan(*cfg, *p, expect)) {
        delete p;
        return fail(NSM_ERR_UNSUPPORTED, "layers=%d exceeds the supported depth", cfg->layers);
    }
    // name-set check as load_network (network.py:271-273)
    std::map<std::string, int> given;
    for (int i = 0; i < n_tensors; ++i) given[names[i]] = i;
    bool same = given.size() == expect.size() && (int)given.size() == n_tensors;
    for (auto& kv : expect) same = same && given.count(kv.first);
    if (!same) {
        delete p;
        return fail(NSM_ERR_FORMAT, "checkpoint parameters do not match config");
    }
    // shapes, then one device block: fp32 weights + biases (+ packed tiles)
    std::vector<char> blob;
    std::map<std::string, size_t> off;
    for (auto& kv : expect) {
        const int i = given[kv.first];
        const Spec& s = kv.second;
        const bool is_w = s.k != 0;
        const int want_nd = is_w ? 4 : 1;
        bool ok = ndims[i] == want_nd;
        if (ok && is_w)
            ok = dims[i][0] == s.cout && dims[i][1] == s.cin && dims[i][2] == s.k && dims[i][3] == s.k;
        else if (ok)
            ok = dims[i][0] == s.cout;
        if (!ok) {
            delete p;
            return fail(NSM_ERR_SHAPE, "parameter %s has the wrong shape for the config", kv.first.c_str());
        }
        const size_t cnt = is_w ? (size_t)s.cout * s.cin * s.k * s.k : (size_t)s.cout;
        off[kv.first] = blob.size();
        blob.resize(blob.size() + ((cnt * 4 + 255) / 256) * 256);
        memcpy(blob.data() + off[kv.first], host_data[i], cnt * 4);
        p->n_params += (int64_t)cnt;
    }
    size_t pk_off = 0;
    if (act_dtype != NSM_F32) {
        // packed tensor-core tiles are laid out after the fp32 tensors
        for (auto& kv : expect) {
            ConvW* c = conv_by_name(*p, kv.first.substr(0, kv.first.size() - 2));
            if (kv.second.k) c->w32 = (const float*)(blob.data() + off[kv.first]);
            else c->b32 = (const float*)(blob.data() + off[kv.first]);
        }
        nsm_status st = pack_f16(*p, blob, pk_off);
        if (st != NSM_OK) {
            delete p;
            return st;
        }
    }
    void* dev = nullptr;
    cudaError_t e = cudaMalloc(&dev, blob.size());
    if (e == cudaSuccess) e = cudaMemcpy(dev, blob.data(), blob.size(), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        if (dev) cudaFree(dev);
        delete p;
        return fail(NSM_ERR_CUDA, "plan upload: %s", cudaGetErrorString(e));
    }
    p->dev = dev;
    p->dev_bytes = blob.size();
    cudaGetDevice(&p->device);
    for (auto& kv : expect) {
        ConvW* c = conv_by_name(*p, kv.first.substr(0, kv.first.size() - 2));
        const float* d = (const float*)((char*)dev + off[kv.first]);
        if (kv.second.k) c->w32 = d;
        else c->b32 = d;
    }
    if (act_dtype != NSM_F32) {
        // rebase the packed pointers (pack_f16 stored host-blob offsets)
        auto rebase = [&](ConvW& c) {
            if (c.present()) c.wpk = (const char*)dev + (size_t)(uintptr_t)c.wpk;
        };
        for (int j = 0; j < p->nlev; ++j) {
            rebase(p->lev[j].enc3);
            rebase(p->lev[j].enc1);
            rebase(p->lev[j].dec3);
            rebase(p->lev[j].dec1);
        }
        rebase(p->head);
        rebase(p->d0p3);
        rebase(p->d0p1);
        rebase(p->d0ph);
    }
    *out_plan = reinterpret_cast<nsm_plan*>(p);
    return NSM_OK;
}

void nsm_plan_destroy(nsm_plan* plan) {
    Plan* p = reinterpret_cast<Plan*>(plan);
    if (!p) return;
    if (p->dev) cudaFree(p->dev);
    delete p;
}

nsm_status nsm_plan_info(const nsm_plan* plan, nsm_net_config* cfg, nsm_dtype* act,
                         int64_t* n_params) {
    const Plan* p = reinterpret_cast<const Plan*>(plan);
    if (!p) return fail(NSM_ERR_ARG, "null plan");
    if (cfg) *cfg = p->cfg;
    if (act) *act = p->act;
    if (n_params) *n_params = p->n_params;
    return NSM_OK;
}

size_t nsm_workspace_size(const nsm_plan* plan, int32_t n, int32_t h, int32_t w) {
    const Plan* p = reinterpret_cast<const Plan*>(plan);
    if (!p || n <= 0 || h <= 0 || w <= 0) return 0;
    const int m = 1 << (p->cfg.layers - 1);
    const int hp = round_up(h, m), wp = round_up(w, m);
    // 16-bit plans run every entry point on the chunked 16-bit kernels, whose
    // workspace is bounded by the chunk, not by n
    if (p->act != NSM_F32 && f16_supported(*p)) return infer_f16_workspace(*p, n, h, w);
    size_t a = forward_any_workspace(*p, n, hp, wp);
    size_t b = infer_f32_workspace(*p, n, h, w);
    return std::max(a, b);
}

nsm_status nsm_features(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                        const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                        float* out_planes, int32_t* texel_idx, int64_t* first_bad, void* stream) {
    clear_error();
    if (!g || !sm || !frames || !out_planes || !first_bad || !g->d || !g->position)
        return fail(NSM_ERR_ARG, "nsm_features: null argument");
    if (n <= 0 || h <= 0 || w <= 0) return fail(NSM_ERR_ARG, "nsm_features: empty batch");
    if (g->dtype != NSM_F32 && g->dtype != NSM_F64)
        return fail(NSM_ERR_ARG, "G-buffer planes must be F32 or F64");
    if (!(g->z_f && g->c_e && g->c_c) && !g->normal)
        return fail(NSM_ERR_ARG, "normal plane needed to derive z_f/c_e/c_c");
    if (nsm_status s = check_frames(frames, n, h, w, sm_stride)) return s;
    return launch_features(g, sm, sm_stride, frames, n, h, w, h, w, out_planes, texel_idx,
                           first_bad, (cudaStream_t)stream);
}

nsm_status nsm_blocker_plane(const nsm_gbuffer* g, const float* sm, int64_t sm_stride,
                             const nsm_frame* frames, int32_t n, int32_t h, int32_t w, int32_t radius,
                             float* out, int64_t* first_bad, void* stream) {
    clear_error();
    if (!g || !sm || !frames || !out || !first_bad || !g->d || !g->position)
        return fail(NSM_ERR_ARG, "nsm_blocker_plane: null argument");
    if (n <= 0 || h <= 0 || w <= 0 || radius <= 0) return fail(NSM_ERR_ARG, "nsm_blocker_plane: bad size");
    if (g->dtype != NSM_F32 && g->dtype != NSM_F64) return fail(NSM_ERR_ARG, "G-buffer planes must be F32 or F64");
    if (nsm_status s = check_frames(frames, n, h, w, sm_stride)) return s;
    return launch_blocker(g, sm, sm_stride, frames, n, h, w, radius, out, first_bad, (cudaStream_t)stream);
}

nsm_status nsm_features5(const nsm_gbuffer* g, const float* sm, int64_t sm_stride, const nsm_frame* frames,
                         int32_t n, int32_t h, int32_t w, float* out_planes, int32_t* texel_idx,
                         int64_t* first_bad, void* stream) {
    clear_error();
    if (!g || !sm || !frames || !out_planes || !first_bad || !g->d || !g->normal || !g->position)
        return fail(NSM_ERR_ARG, "nsm_features5: null argument");
    if (n <= 0 || h <= 0 || w <= 0) return fail(NSM_ERR_ARG, "nsm_features5: empty batch");
    if (nsm_status s = check_frames(frames, n, h, w, sm_stride)) return s;
    cudaStream_t st = (cudaStream_t)stream;
    launch_fill_i64(first_bad, n, INT64_MAX, st);
    for (int f0 = 0; f0 < n; f0 += NSM_MAX_FRAMES_PER_LAUNCH) {
        const int nf = std::min(n - f0, NSM_MAX_FRAMES_PER_LAUNCH);
        nsm_gbuffer gc = *g;
        gc.d = (const float*)g->d + (int64_t)f0 * g->frame_stride;
        gc.normal = (const float*)g->normal + (int64_t)f0 * 3 * g->frame_stride;
        gc.position = (const float*)g->position + (int64_t)f0 * 3 * g->frame_stride;
        nsm_status s = launch_feat5(&gc, sm + f0 * sm_stride, sm_stride, frames + f0, nf, h, w, 0, 0,
                                    out_planes + (int64_t)f0 * 5 * h * w, 2, first_bad + f0,
                                    texel_idx ? texel_idx + (int64_t)f0 * 2 * h * w : nullptr, st,
                                    g_feat5_dbg ? g_feat5_dbg + (int64_t)f0 * h * w * 4 : nullptr);
        if (s != NSM_OK) return s;
    }
    return check_stream_err();
}

nsm_status nsm_forward(const nsm_plan* plan, const float* x, int32_t n, int32_t h, int32_t w,
                       float* y, void* workspace, size_t ws_bytes, void* stream) {
    clear_error();
    const Plan* p = reinterpret_cast<const Plan*>(plan);
    if (!p || !x || !y || !workspace) return fail(NSM_ERR_ARG, "nsm_forward: null argument");
    if (n <= 0) return fail(NSM_ERR_ARG, "nsm_forward: empty batch");
    const int f = 1 << (p->cfg.layers - 1);
    // network.forward (network.py:169-173)
    if (h <= 0 || w <= 0 || h % f || w % f)
        return fail(NSM_ERR_SHAPE, "spatial dims %dx%d must be divisible by %d", h, w, f);
    if (nsm_status s = check_device(*p)) return s;
    if (p->act == NSM_F32)
        return forward_f32(*p, x, n, h, w, y, workspace, ws_bytes, (cudaStream_t)stream);
    if (!f16_supported(*p))   // the generic layer-by-layer 16-bit path
        return forward_gen16(*p, x, n, h, w, y, workspace, ws_bytes, (cudaStream_t)stream);
    return forward_f16(*p, x, n, h, w, y, workspace, ws_bytes, (cudaStream_t)stream);
}

nsm_status nsm_infer(const nsm_plan* plan, const nsm_gbuffer* g, const float* sm,
                     int64_t sm_stride, const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                     void* y, nsm_dtype y_dtype, int64_t* first_bad, void* workspace,
                     size_t ws_bytes, void* stream) {
    return nsm_infer_ex(plan, g, sm, sm_stride, frames, n, h, w, y, y_dtype, first_bad, nullptr, workspace,
                        ws_bytes, stream);
}

nsm_status nsm_infer_ex(const nsm_plan* plan, const nsm_gbuffer* g, const float* sm,
                        int64_t sm_stride, const nsm_frame* frames, int32_t n, int32_t h, int32_t w,
                        void* y, nsm_dtype y_dtype, int64_t* first_bad, int32_t* texel_idx, void* workspace,
                        size_t ws_bytes, void* stream) {
    clear_error();
    const Plan* p = reinterpret_cast<const Plan*>(plan);
    if (!p || !g || !sm || !frames || !y || !first_bad || !workspace || !g->d || !g->position)
        return fail(NSM_ERR_ARG, "nsm_infer: null argument");
    if (n <= 0 || h <= 0 || w <= 0) return fail(NSM_ERR_ARG, "nsm_infer: empty batch");
    if (y_dtype != NSM_F32 && y_dtype != NSM_F16) return fail(NSM_ERR_ARG, "y_dtype must be F32 or F16");
    // the feature pass produces the 4 reference planes, plus the
    // blocker-search penumbra plane for in_channels = 5 nets (16-bit plans)
    if (p->cfg.in_channels == 5 && (p->act == NSM_F32 || !f16_supported(*p)))
        return fail(NSM_ERR_UNSUPPORTED, "the fused 5-plane feature pass runs with the default 16-bit net; "
                                         "use nsm_features5 + nsm_forward");
    if (p->cfg.in_channels != 4 && p->cfg.in_channels != 5)
        return fail(NSM_ERR_SHAPE, "input has 4 channels, config wants %d", p->cfg.in_channels);
    if (g->dtype != NSM_F32 && g->dtype != NSM_F64)
        return fail(NSM_ERR_ARG, "G-buffer planes must be F32 or F64");
    if (!(g->z_f && g->c_e && g->c_c) && !g->normal)
        return fail(NSM_ERR_ARG, "normal plane needed to derive z_f/c_e/c_c");
    if (nsm_status s = check_frames(frames, n, h, w, sm_stride)) return s;
    if (nsm_status s = check_device(*p)) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if (p->act != NSM_F32 && f16_supported(*p)) {
        return infer_f16(*p, g, sm, sm_stride, frames, n, h, w, y, y_dtype, first_bad, texel_idx,
                         workspace, ws_bytes, st);
    }
    if (ws_bytes < infer_f32_workspace(*p, n, h, w))
        return fail(NSM_ERR_ARG, "workspace too small");
    const int m = 1 << (p->cfg.layers - 1);
    const int hp = round_up(h, m), wp = round_up(w, m);
    float* feat = (float*)workspace;
    float* yfull = feat + (size_t)n * 4 * hp * wp;
    char* rest = (char*)(yfull + (size_t)n * hp * wp);
    rest = (char*)(((uintptr_t)rest + 255) & ~(uintptr_t)255);
    if (texel_idx && (hp != h || wp != w))
        return fail(NSM_ERR_UNSUPPORTED, "texel_idx on an fp32 plan needs h, w divisible by %d", m);
    nsm_status s = launch_features(g, sm, sm_stride, frames, n, h, w, hp, wp, feat, texel_idx,
                                   first_bad, st);
    if (s != NSM_OK) return s;
    const bool direct = (hp == h && wp == w && y_dtype == NSM_F32);
    float* yo = direct ? (float*)y : yfull;
    const size_t rest_bytes = ws_bytes - (size_t)(rest - (char*)workspace);
    s = p->act == NSM_F32 ? forward_f32(*p, feat, n, hp, wp, yo, rest, rest_bytes, st)
                          : forward_gen16(*p, feat, n, hp, wp, yo, rest, rest_bytes, st);
    if (s != NSM_OK) return s;
    if (!direct) {
        const int64_t tot = (int64_t)n * h * w;
        const int grid = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
        NSM_PROF("crop_kernel", st);
        crop_kernel<<<grid, 256, 0, st>>>(yfull, hp, wp, h, w, n, y, y_dtype == NSM_F16);
    }
    return check_stream_err();
}

nsm_status nsm_render_gbuffer(const double* prims, int32_t n_prims, const nsm_camera* cam,
                              float* d, float* normal, float* position, void* stream) {
    clear_error();
    if (!prims || !cam || !d || !normal || !position || n_prims <= 0)
        return fail(NSM_ERR_ARG, "nsm_render_gbuffer: bad argument");
    return launch_render_gbuffer(prims, n_prims, cam, d, normal, position, (cudaStream_t)stream);
}

nsm_status nsm_render_shadowmap(const double* prims, int32_t n_prims, const nsm_emitter_view* view,
                                float* depth, void* stream) {
    clear_error();
    if (!prims || !view || !depth || n_prims <= 0)
        return fail(NSM_ERR_ARG, "nsm_render_shadowmap: bad argument");
    return launch_render_shadowmap(prims, n_prims, view, depth, (cudaStream_t)stream);
}

nsm_status nsm_motion_vectors(const nsm_gbuffer* g, const nsm_camera* cams, int32_t t_frames,
                              int32_t h, int32_t w, double* vec, uint8_t* valid, void* stream) {
    clear_error();
    if (!g || !cams || !vec || !valid || !g->d || !g->normal || !g->position)
        return fail(NSM_ERR_ARG, "nsm_motion_vectors: null argument");
    if (t_frames < 2 || h <= 0 || w <= 0) return fail(NSM_ERR_ARG, "nsm_motion_vectors: need >= 2 frames");
    if (g->dtype != NSM_F32 && g->dtype != NSM_F64)
        return fail(NSM_ERR_ARG, "G-buffer planes must be F32 or F64");
    for (int k = 0; k < t_frames - 1; ++k)
        if (cams[k].height != h || cams[k].width != w)  // raster.py:337-338
            return fail(NSM_ERR_ARG, "motion vectors need equal resolutions");
    return launch_motion(g, cams, t_frames, h, w, vec, valid, (cudaStream_t)stream);
}

nsm_status nsm_temporal_instability(const float* vis, const double* vec, const uint8_t* valid,
                                    int32_t t_frames, int32_t h, int32_t w, double alpha, double* acc,
                                    uint64_t* count, void* stream) {
    clear_error();
    if (!vis || !vec || !valid || !acc || !count) return fail(NSM_ERR_ARG, "nsm_temporal_instability: null argument");
    if (t_frames < 2) return fail(NSM_ERR_ARG, "need at least two frames");  // analysis.py:353-354
    if (h <= 0 || w <= 0) return fail(NSM_ERR_ARG, "nsm_temporal_instability: empty frames");
    return launch_instability(vis, vec, valid, t_frames, h, w, alpha, acc, (unsigned long long*)count,
                              (cudaStream_t)stream);
}

}  // extern "C"
