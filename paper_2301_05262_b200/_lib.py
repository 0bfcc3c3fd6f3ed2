"""ctypes binding of the C-ABI library (include/nsm.h).

The library is the product: there is no Python or CPU fallback. Importing
this module loads ``libnsm.so`` (built in-tree by ``build.py``) and raises
immediately if it is missing; every call raises the reference's exception
type for the returned status code.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnsm.so")

NSM_OK, NSM_ERR_ARG, NSM_ERR_SHAPE, NSM_ERR_FRUSTUM, NSM_ERR_FORMAT, NSM_ERR_CUDA, \
    NSM_ERR_UNSUPPORTED = range(7)
NSM_F32, NSM_F16, NSM_BF16, NSM_F64 = range(4)
MAX_FRAMES_PER_LAUNCH = 8
ABI_VERSION = 2
BUILD_EXPERIMENTS = 1
INT64_MAX = (1 << 63) - 1


class FrustumError(RuntimeError):
    """A covered camera pixel projects outside the emitter frustum
    (raster.py:60-61)."""


class FormatError(ValueError):
    """Corrupt or mismatching binary file / checkpoint (fileio.py:22-23)."""


class NetConfig(C.Structure):
    _fields_ = [("layers", C.c_int32), ("base_channels", C.c_int32),
                ("in_channels", C.c_int32), ("use_space_to_depth", C.c_int32),
                ("channel_cap", C.c_int32)]


class EmitterViewC(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("forward", C.c_double * 3),
                ("up", C.c_double * 3), ("right", C.c_double * 3),
                ("tan_half", C.c_double), ("height", C.c_int32), ("width", C.c_int32)]


class CameraC(C.Structure):
    _fields_ = [("position", C.c_double * 3), ("forward", C.c_double * 3),
                ("up", C.c_double * 3), ("fov_y", C.c_double),
                ("height", C.c_int32), ("width", C.c_int32)]


class FrameC(C.Structure):
    _fields_ = [("camera", CameraC), ("view", EmitterViewC),
                ("emitter_center", C.c_double * 3), ("size_index", C.c_double),
                ("bias", C.c_double)]


class GBufferC(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("d", C.c_void_p), ("normal", C.c_void_p),
                ("position", C.c_void_p), ("z_f", C.c_void_p), ("c_e", C.c_void_p),
                ("c_c", C.c_void_p), ("coverage", C.c_void_p), ("frame_stride", C.c_int64)]


class PlanHandle(C.Structure):
    pass


_EXPORTS = {
    "nsm_plan_create": (C.c_int, [C.POINTER(NetConfig), C.c_int32, C.POINTER(C.c_char_p),
                                  C.POINTER(C.c_void_p), C.POINTER(C.c_int32),
                                  C.POINTER(C.POINTER(C.c_int32)), C.c_int32,
                                  C.POINTER(C.POINTER(PlanHandle))]),
    "nsm_plan_destroy": (None, [C.POINTER(PlanHandle)]),
    "nsm_plan_info": (C.c_int, [C.POINTER(PlanHandle), C.POINTER(NetConfig),
                                C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "nsm_workspace_size": (C.c_size_t, [C.POINTER(PlanHandle), C.c_int32, C.c_int32, C.c_int32]),
    "nsm_features": (C.c_int, [C.POINTER(GBufferC), C.c_void_p, C.c_int64, C.POINTER(FrameC),
                               C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]),
    "nsm_blocker_plane": (C.c_int, [C.POINTER(GBufferC), C.c_void_p, C.c_int64, C.POINTER(FrameC),
                                    C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p]),
    "nsm_features5": (C.c_int, [C.POINTER(GBufferC), C.c_void_p, C.c_int64, C.POINTER(FrameC),
                                C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p]),
    "nsm_forward": (C.c_int, [C.POINTER(PlanHandle), C.c_void_p, C.c_int32, C.c_int32,
                              C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "nsm_infer": (C.c_int, [C.POINTER(PlanHandle), C.POINTER(GBufferC), C.c_void_p, C.c_int64,
                            C.POINTER(FrameC), C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                            C.c_int32, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "nsm_infer_ex": (C.c_int, [C.POINTER(PlanHandle), C.POINTER(GBufferC), C.c_void_p, C.c_int64,
                               C.POINTER(FrameC), C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                               C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                               C.c_void_p]),
    "nsm_render_gbuffer": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(CameraC), C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p]),
    "nsm_render_shadowmap": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(EmitterViewC),
                                       C.c_void_p, C.c_void_p]),
    "nsm_motion_vectors": (C.c_int, [C.POINTER(GBufferC), C.POINTER(CameraC), C.c_int32, C.c_int32,
                                     C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p]),
    "nsm_temporal_instability": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                           C.c_int32, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "nsm_launch_count": (C.c_int64, []),
    "nsm_profile_enable": (None, [C.c_int32]),
    "nsm_profile_report": (C.c_int32, [C.c_char_p, C.c_size_t]),
    "nsm_last_error": (C.c_char_p, []),
    "nsm_abi_version": (C.c_int32, []),
    "nsm_build_flags": (C.c_int32, []),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _EXPORTS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
if lib.nsm_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH} has ABI {lib.nsm_abi_version()}, this binding wants {ABI_VERSION}: rebuild")


def experiment_build() -> bool:
    """True when libnsm.so was built with -DNSM_EXPERIMENTS (tools/ only)."""
    return bool(lib.nsm_build_flags() & BUILD_EXPERIMENTS)


def check(status: int, what: str = "") -> None:
    """Raise the reference exception type for a non-OK status."""
    if status == NSM_OK:
        return
    msg = lib.nsm_last_error().decode() or what
    if status in (NSM_ERR_ARG, NSM_ERR_SHAPE):
        raise ValueError(msg)
    if status == NSM_ERR_FRUSTUM:
        raise FrustumError(msg)
    if status == NSM_ERR_FORMAT:
        raise FormatError(msg)
    if status == NSM_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def _vec(v):
    return (C.c_double * 3)(*[float(a) for a in v])


def view_c(view) -> EmitterViewC:
    h, w = view.resolution
    return EmitterViewC(_vec(view.position), _vec(view.forward), _vec(view.up), _vec(view.right),
                        float(view.tan_half), int(h), int(w))


def camera_c(cam) -> CameraC:
    h, w = cam.resolution
    return CameraC(_vec(cam.position), _vec(cam.forward), _vec(cam.up), float(cam.fov_y),
                   int(h), int(w))


def frames_c(items) -> C.Array:
    """items: iterable of (camera, view, emitter_center, size_index, bias)."""
    items = list(items)
    arr = (FrameC * len(items))()
    for i, (cam, view, center, s, b) in enumerate(items):
        arr[i] = FrameC(camera_c(cam), view_c(view), _vec(center), float(s), float(b))
    return arr


def profile_report() -> dict:
    """{kernel name: (launches, total_ms)} of the traced launches since the
    last report (nsm_profile_report)."""
    buf = C.create_string_buffer(1 << 16)
    lib.nsm_profile_report(buf, len(buf))
    out = {}
    for line in buf.value.decode().splitlines():
        name, cnt, ms = line.split()
        out[name] = (int(cnt), float(ms))
    return out


def stream_ptr(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)
