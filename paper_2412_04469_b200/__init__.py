"""QUEEN per-frame decode -> apply -> 3D-GS splat on B200 (sm_100a).

Thin Python binding over the C-ABI library ``libqueen.so`` (include/queen.h).
Argument marshalling only: every step of the path runs in the library's CUDA
kernels.  PyTorch provides device memory and streams.  There is NO CPU fallback:
if the extension is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# QUEEN_LIB_PATH: load an experiment build (tools/variants.py) instead of the in-tree library
LIB_PATH = os.environ.get("QUEEN_LIB_PATH") or os.path.join(_HERE, "libqueen.so")

QUEEN_OK = 0
QUEEN_WARN_NONFINITE = 1
STATUS = {0: "QUEEN_OK", -1: "QUEEN_ERR_INVALID_ARG", -2: "QUEEN_ERR_SHAPE", -3: "QUEEN_ERR_INDEX",
          -4: "QUEEN_ERR_LATENT_RANGE", -5: "QUEEN_ERR_CAPACITY", -6: "QUEEN_ERR_CUDA", -7: "QUEEN_ERR_TIMEOUT",
          1: "QUEEN_WARN_NONFINITE"}
QUEEN_LAT_INT8, QUEEN_LAT_F32 = 0, 1
QUEEN_POS_COO, QUEEN_POS_GATES, QUEEN_POS_NONE = 0, 1, 2
QUEEN_MAX_VIEWS = 64
QUEEN_OPT_BLEND_NOMASK, QUEEN_OPT_BLEND_GRID_ORDER = 1, 2

# exported C symbols (include/queen.h); tests check the library exports every one
EXPORTS = ["queen_create", "queen_destroy", "queen_last_error", "queen_version", "queen_workspace_size",
           "queen_set_workspace", "queen_check", "queen_decode_residuals", "queen_apply_frame", "queen_project",
           "queen_bin_sort", "queen_rasterize", "queen_render_views", "queen_blend_counts",
           "queen_profile_enable", "queen_profile_read", "queen_wait_binned", "queen_wait_projected", "queen_set_blend_stream",
           "queen_wait_rendered", "queen_entropy_encode",
           "queen_entropy_decode", "queen_entropy_decode_frame", "queen_render_mask",
           "queen_densify", "queen_rasterize_rgb8", "queen_render_views_rgb8",
           "queen_rasterize_backward", "queen_project_backward", "queen_decode_backward", "queen_set_options",
           "queen_rasterize_f16", "queen_render_views_f16", "queen_set_sh_rest",
           "queen_rasterize_rgb10", "queen_render_views_rgb10"]
STAGES = ["apply", "project", "compact", "depth_sort", "bucket", "emit", "ranges", "blend", "entropy", "blend_order"]


class QueenError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


# ---------------------------------------------------------------- C structs
class QueenGaussians(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_pad", C.c_int32), ("sh_degree", C.c_int32), ("planes", C.c_void_p)]


class QueenPacket(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_pad", C.c_int32), ("sh_degree", C.c_int32), ("lat_dim", C.c_int32 * 5),
                ("latent_kind", C.c_int32), ("latents", C.c_void_p), ("decoders", C.c_void_p),
                ("pos_kind", C.c_int32), ("k", C.c_int32), ("k_dev", C.c_void_p), ("pos_idx", C.c_void_p),
                ("pos_val", C.c_void_p), ("log_alpha", C.c_void_p), ("pos_pregate", C.c_void_p),
                ("tau", C.c_float), ("gamma0", C.c_float), ("gamma1", C.c_float)]


class QueenCamera(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float), ("R", C.c_float * 9),
                ("t", C.c_float * 3), ("C", C.c_float * 3), ("limx", C.c_float), ("limy", C.c_float),
                ("near_z", C.c_float), ("width", C.c_int32), ("height", C.c_int32)]


class QueenProj(C.Structure):
    _fields_ = [("n_pad", C.c_int32), ("rec", C.c_void_p), ("depth", C.c_void_p), ("tiles", C.c_void_p),
                ("rect", C.c_void_p)]


class QueenBins(C.Structure):
    _fields_ = [("keys_cap", C.c_int64), ("keys", C.c_void_p), ("keys_alt", C.c_void_p), ("vals", C.c_void_p),
                ("vals_alt", C.c_void_p), ("ranges", C.c_void_p), ("K", C.c_void_p),
                ("sorted_in_alt", C.c_int32)]


assert C.sizeof(QueenCamera) == 96


_lib = None


def lib() -> C.CDLL:
    """Load libqueen.so (fails loudly if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libqueen.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        p, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "queen_create": (i32, [C.c_int, C.POINTER(p)]),
            "queen_destroy": (None, [p]),
            "queen_last_error": (C.c_char_p, [p]),
            "queen_version": (C.c_char_p, []),
            "queen_workspace_size": (i32, [i32, i32, i32, i32, i64, C.POINTER(C.c_size_t)]),
            "queen_set_workspace": (i32, [p, p, C.c_size_t, i32, i32, i32, i32, i64]),
            "queen_check": (i32, [p, p, C.POINTER(C.c_int64)]),
            "queen_decode_residuals": (i32, [p, C.POINTER(QueenPacket), p, p, p, p, p, p]),
            "queen_apply_frame": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenPacket), p]),
            "queen_project": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenCamera), i32, C.POINTER(QueenProj), p]),
            "queen_bin_sort": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenCamera), i32, C.POINTER(QueenBins), p]),
            "queen_rasterize": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenBins), C.POINTER(QueenCamera), i32,
                                      C.POINTER(C.c_float), p, p, p]),
            "queen_render_views": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenCamera), i32,
                                         C.POINTER(C.c_float), p, p, p]),
            "queen_blend_counts": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenBins), C.POINTER(QueenCamera), i32,
                                         p, p, p]),
            "queen_profile_enable": (i32, [p, i32]),
            "queen_set_options": (i32, [p, i32]),
            "queen_set_sh_rest": (i32, [p, C.POINTER(QueenGaussians), p, i32, p, p]),
            "queen_decode_backward": (i32, [p, C.POINTER(QueenPacket), p, p, p, p, p, p]),
            "queen_rasterize_backward": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenBins), C.POINTER(QueenCamera),
                                               i32, C.POINTER(C.c_float), p, p, p]),
            "queen_project_backward": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenCamera), i32, p, p, p]),
            "queen_rasterize_rgb8": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenBins), C.POINTER(QueenCamera), i32,
                                           C.POINTER(C.c_float), p, p, p]),
            "queen_render_views_rgb8": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenCamera), i32,
                                              C.POINTER(C.c_float), p, p, p]),
            "queen_rasterize_f16": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenBins), C.POINTER(QueenCamera), i32,
                                           C.POINTER(C.c_float), p, p, p]),
            "queen_render_views_f16": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenCamera), i32,
                                              C.POINTER(C.c_float), p, p, p]),
            "queen_rasterize_rgb10": (i32, [p, C.POINTER(QueenProj), C.POINTER(QueenBins), C.POINTER(QueenCamera), i32,
                                           C.POINTER(C.c_float), p, p, p]),
            "queen_render_views_rgb10": (i32, [p, C.POINTER(QueenGaussians), C.POINTER(QueenCamera), i32,
                                              C.POINTER(C.c_float), p, p, p]),
            "queen_densify": (i32, [p, C.POINTER(QueenGaussians), p, i32, p, i32, C.POINTER(QueenGaussians), p]),
            "queen_render_mask": (i32, [p, C.POINTER(QueenGaussians), p, i32, p, C.POINTER(QueenCamera), i32, C.c_float,
                                        i32, p, p]),
            "queen_wait_binned": (i32, [p, p]),
            "queen_wait_projected": (i32, [p, p]),
            "queen_set_blend_stream": (i32, [p, p]),
            "queen_wait_rendered": (i32, [p, p]),
            "queen_entropy_encode": (i32, [p, i32, i32, i32, p, C.c_size_t, C.POINTER(C.c_size_t)]),
            "queen_entropy_decode": (i32, [p, p, C.c_int64, i32, i32, i32, p, p]),
            "queen_entropy_decode_frame": (i32, [p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                                 i32, i32, p, p]),
            "queen_profile_read": (i32, [p, C.POINTER(C.c_double), C.POINTER(C.c_int64), i32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


# ---------------------------------------------------------------- helpers
def _ptr(t) -> int | None:
    if t is None:
        return None
    import torch
    if isinstance(t, torch.Tensor):
        if not t.is_cuda:
            raise ValueError("libqueen takes CUDA tensors (no CPU fallback)")
        if not t.is_contiguous():
            raise ValueError("tensors must be contiguous")
        return t.data_ptr()
    return int(t)


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream if hasattr(s, "cuda_stream") else int(s)


def camera_struct(cam) -> QueenCamera:
    """harness.synth.Camera (or anything with the same attributes) -> QueenCamera."""
    c = QueenCamera()
    c.fx, c.fy, c.cx, c.cy = cam.fx, cam.fy, cam.cx, cam.cy
    c.R[:] = [float(x) for x in np.asarray(cam.R, np.float32).reshape(-1)]
    c.t[:] = [float(x) for x in np.asarray(cam.t, np.float32).reshape(-1)]
    c.C[:] = [float(x) for x in np.asarray(cam.C, np.float32).reshape(-1)]
    c.limx, c.limy, c.near_z = cam.limx, cam.limy, cam.near
    c.width, c.height = cam.width, cam.height
    return c


def camera_array(cams):
    arr = (QueenCamera * len(cams))()
    for j, cam in enumerate(cams):
        arr[j] = camera_struct(cam)
    return arr


class Context:
    """One libqueen context on one device, with its torch-allocated workspace."""

    def __init__(self, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libqueen needs a CUDA device (B200); there is no CPU fallback")
        self.device = device
        self._h = C.c_void_p()
        st = lib().queen_create(device, C.byref(self._h))
        if st != QUEEN_OK:
            raise QueenError(st, "queen_create")
        self.ws = None
        self.shape = None

    @property
    def handle(self):
        return self._h

    def last_error(self) -> str:
        return lib().queen_last_error(self._h).decode()

    def _chk(self, st: int, what: str):
        if st != QUEEN_OK:
            raise QueenError(st, f"{what}: {self.last_error()}")

    def set_workspace(self, n_pad: int, n_views: int, width: int, height: int, keys_cap: int):
        import torch
        nbytes = C.c_size_t()
        st = lib().queen_workspace_size(n_pad, n_views, width, height, int(keys_cap), C.byref(nbytes))
        self._chk(st, "queen_workspace_size")
        self.ws = torch.empty(int(nbytes.value) + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        base = self.ws.data_ptr()
        aligned = (base + 255) // 256 * 256
        st = lib().queen_set_workspace(self._h, C.c_void_p(aligned), int(nbytes.value), n_pad, n_views, width, height,
                                       int(keys_cap))
        self._chk(st, "queen_set_workspace")
        self.shape = (n_pad, n_views, width, height, int(keys_cap))

    def check(self, stream=None, allow_warn: bool = True) -> tuple[int, int]:
        info = C.c_int64(0)
        st = lib().queen_check(self._h, C.c_void_p(_stream(stream)), C.byref(info))
        if st < 0 or (st > 0 and not allow_warn):
            raise QueenError(st, f"queen_check: {self.last_error()} (info={info.value})")
        return st, int(info.value)

    def check_status(self, stream=None) -> tuple[int, int]:
        info = C.c_int64(0)
        st = lib().queen_check(self._h, C.c_void_p(_stream(stream)), C.byref(info))
        return st, int(info.value)

    def set_options(self, opts: int):
        self._chk(lib().queen_set_options(self._h, int(opts)), "queen_set_options")

    def profile(self, enable: bool = True):
        self._chk(lib().queen_profile_enable(self._h, 1 if enable else 0), "queen_profile_enable")

    def profile_read(self, reset: bool = True) -> dict:
        ms = (C.c_double * len(STAGES))()
        ln = (C.c_int64 * len(STAGES))()
        self._chk(lib().queen_profile_read(self._h, ms, ln, 1 if reset else 0), "queen_profile_read")
        return {STAGES[i]: (float(ms[i]), int(ln[i])) for i in range(len(STAGES))}

    def __del__(self):
        try:
            if self._h:
                lib().queen_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------- C-ABI mirrors
def gaussians_struct(planes, n: int, sh_degree: int) -> QueenGaussians:
    g = QueenGaussians()
    g.n, g.n_pad, g.sh_degree, g.planes = n, planes.shape[1], sh_degree, _ptr(planes)
    return g


def packet_struct(*, n, n_pad, sh_degree, lat_dim, latents, decoders, latent_kind=QUEEN_LAT_INT8,
                  pos_kind=QUEEN_POS_COO, k=0, k_dev=None, pos_idx=None, pos_val=None, log_alpha=None,
                  pos_pregate=None, gate=(0.3, -0.5, 1.01)) -> QueenPacket:
    p = QueenPacket()
    p.n, p.n_pad, p.sh_degree = n, n_pad, sh_degree
    p.lat_dim[:] = list(lat_dim)
    p.latent_kind = latent_kind
    p.latents, p.decoders = _ptr(latents), _ptr(decoders)
    p.pos_kind, p.k = pos_kind, int(k)
    p.k_dev = _ptr(k_dev)
    p.pos_idx, p.pos_val = _ptr(pos_idx), _ptr(pos_val)
    p.log_alpha, p.pos_pregate = _ptr(log_alpha), _ptr(pos_pregate)
    p.tau, p.gamma0, p.gamma1 = (float(x) for x in gate)
    return p


def queen_decode_residuals(ctx: Context, pkt: QueenPacket, resid_out=None, q_out=None, coo_idx_out=None,
                           coo_val_out=None, k_out=None, stream=None):
    st = lib().queen_decode_residuals(ctx.handle, C.byref(pkt), _ptr(resid_out), _ptr(q_out), _ptr(coo_idx_out),
                                      _ptr(coo_val_out), _ptr(k_out), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_decode_residuals")


def queen_apply_frame(ctx: Context, scene: QueenGaussians, pkt: QueenPacket, stream=None):
    st = lib().queen_apply_frame(ctx.handle, C.byref(scene), C.byref(pkt), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_apply_frame")


def proj_struct(rec, depth, tiles, rect) -> QueenProj:
    pj = QueenProj()
    pj.n_pad = rec.shape[1]
    pj.rec, pj.depth, pj.tiles, pj.rect = _ptr(rec), _ptr(depth), _ptr(tiles), _ptr(rect)
    return pj


def bins_struct(keys, keys_alt, vals, vals_alt, ranges, K) -> QueenBins:
    b = QueenBins()
    b.keys_cap = keys.shape[0]
    b.keys, b.keys_alt, b.vals, b.vals_alt = _ptr(keys), _ptr(keys_alt), _ptr(vals), _ptr(vals_alt)
    b.ranges, b.K = _ptr(ranges), _ptr(K)
    b.sorted_in_alt = 0
    return b


def queen_project(ctx: Context, scene: QueenGaussians, cams, proj: QueenProj, stream=None):
    arr = camera_array(cams)
    st = lib().queen_project(ctx.handle, C.byref(scene), arr, len(cams), C.byref(proj), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_project")


def queen_bin_sort(ctx: Context, proj: QueenProj, cams, bins: QueenBins, stream=None):
    arr = camera_array(cams)
    st = lib().queen_bin_sort(ctx.handle, C.byref(proj), arr, len(cams), C.byref(bins), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_bin_sort")


def queen_rasterize(ctx: Context, proj: QueenProj, bins: QueenBins, cams, rgb_out, T_out=None, bg=(0.0, 0.0, 0.0),
                    stream=None):
    arr = camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_rasterize(ctx.handle, C.byref(proj), C.byref(bins), arr, len(cams), bgv, _ptr(rgb_out),
                               _ptr(T_out), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_rasterize")


def queen_render_views(ctx: Context, scene: QueenGaussians, cams, rgb_out, T_out=None, bg=(0.0, 0.0, 0.0),
                       stream=None, cam_array=None):
    arr = cam_array if cam_array is not None else camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_render_views(ctx.handle, C.byref(scene), arr, len(arr), bgv, _ptr(rgb_out), _ptr(T_out),
                                  C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_render_views")


def queen_render_mask(ctx: Context, scene: QueenGaussians, subset_idx, k: int, cams, mask_out, alpha_thresh=1e-3,
                      dilation: int = 48, k_dev=None, stream=None, cam_array=None):
    """NEXT #3: dilated alpha mask of the subset's rendering (queen.h queen_render_mask)."""
    arr = cam_array if cam_array is not None else camera_array(cams)
    st = lib().queen_render_mask(ctx.handle, C.byref(scene), _ptr(subset_idx), int(k), _ptr(k_dev), arr, len(arr),
                                 float(alpha_thresh), int(dilation), _ptr(mask_out), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_render_mask")


def queen_densify(ctx: Context, src: QueenGaussians, rem_idx, n_rem: int, add_attrs, n_add: int, dst: QueenGaussians,
                  stream=None):
    """NEXT #2: dst = src minus the removed columns, plus the binary16 additions (queen.h)."""
    st = lib().queen_densify(ctx.handle, C.byref(src), _ptr(rem_idx), int(n_rem), _ptr(add_attrs), int(n_add),
                             C.byref(dst), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_densify")


def queen_rasterize_rgb8(ctx: Context, proj: QueenProj, bins: QueenBins, cams, rgb8_out, T_out=None,
                         bg=(0.0, 0.0, 0.0), stream=None):
    arr = camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_rasterize_rgb8(ctx.handle, C.byref(proj), C.byref(bins), arr, len(arr), bgv, _ptr(rgb8_out),
                                    _ptr(T_out), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_rasterize_rgb8")


def queen_render_views_rgb8(ctx: Context, scene: QueenGaussians, cams, rgb8_out, T_out=None, bg=(0.0, 0.0, 0.0),
                            stream=None, cam_array=None):
    arr = cam_array if cam_array is not None else camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_render_views_rgb8(ctx.handle, C.byref(scene), arr, len(arr), bgv, _ptr(rgb8_out), _ptr(T_out),
                                       C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_render_views_rgb8")


def queen_rasterize_f16(ctx: Context, proj: QueenProj, bins: QueenBins, cams, f16_out, T_out=None,
                         bg=(0.0, 0.0, 0.0), stream=None):
    arr = camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_rasterize_f16(ctx.handle, C.byref(proj), C.byref(bins), arr, len(arr), bgv, _ptr(f16_out),
                                    _ptr(T_out), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_rasterize_f16")


def queen_render_views_f16(ctx: Context, scene: QueenGaussians, cams, f16_out, T_out=None, bg=(0.0, 0.0, 0.0),
                            stream=None, cam_array=None):
    arr = cam_array if cam_array is not None else camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_render_views_f16(ctx.handle, C.byref(scene), arr, len(arr), bgv, _ptr(f16_out), _ptr(T_out),
                                       C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_render_views_f16")


def queen_rasterize_rgb10(ctx: Context, proj: QueenProj, bins: QueenBins, cams, rgb10_out, T_out=None,
                         bg=(0.0, 0.0, 0.0), stream=None):
    arr = camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_rasterize_rgb10(ctx.handle, C.byref(proj), C.byref(bins), arr, len(arr), bgv, _ptr(rgb10_out),
                                    _ptr(T_out), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_rasterize_rgb10")


def queen_render_views_rgb10(ctx: Context, scene: QueenGaussians, cams, rgb10_out, T_out=None, bg=(0.0, 0.0, 0.0),
                            stream=None, cam_array=None):
    arr = cam_array if cam_array is not None else camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_render_views_rgb10(ctx.handle, C.byref(scene), arr, len(arr), bgv, _ptr(rgb10_out), _ptr(T_out),
                                       C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_render_views_rgb10")


def queen_rasterize_backward(ctx: Context, proj: QueenProj, bins: QueenBins, cams, dL_drgb, grad_rec,
                             bg=(0.0, 0.0, 0.0), stream=None):
    """NEXT #4: dL/d(record) [V][n_pad][9] from dL/d(image) [V][3][H][W] (queen.h)."""
    arr = camera_array(cams)
    bgv = (C.c_float * 3)(*[float(x) for x in bg])
    st = lib().queen_rasterize_backward(ctx.handle, C.byref(proj), C.byref(bins), arr, len(arr), bgv, _ptr(dL_drgb),
                                        _ptr(grad_rec), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_rasterize_backward")


def queen_project_backward(ctx: Context, scene: QueenGaussians, cams, grad_rec, grad_planes, stream=None):
    """NEXT #4: dL/d(raw attributes) [P][n_pad] from dL/d(record) (queen.h)."""
    arr = camera_array(cams)
    st = lib().queen_project_backward(ctx.handle, C.byref(scene), arr, len(arr), _ptr(grad_rec), _ptr(grad_planes),
                                      C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_project_backward")


def queen_decode_backward(ctx: Context, pkt: QueenPacket, grad_planes, grad_decoders=None, grad_latents=None,
                          grad_log_alpha=None, grad_pregate=None, stream=None):
    """NEXT #4: decoder / straight-through latent / gate gradients from dL/dA_t (queen.h)."""
    st = lib().queen_decode_backward(ctx.handle, C.byref(pkt), _ptr(grad_planes), _ptr(grad_decoders),
                                     _ptr(grad_latents), _ptr(grad_log_alpha), _ptr(grad_pregate),
                                     C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_decode_backward")


def queen_entropy_encode(latents: np.ndarray, n: int) -> np.ndarray:
    """Host rANS encode of one category's int8 latent matrix [L][n_pad] -> uint8 QANS stream."""
    lat = np.ascontiguousarray(latents, np.int8)
    L, n_pad = lat.shape
    nb = C.c_size_t(0)
    cap = 2 * L * max(n, 1) + 64 * 1024 + 160 * (L * n // 16384 + 2)
    out = np.zeros(cap, np.uint8)
    st = lib().queen_entropy_encode(lat.ctypes.data_as(C.c_void_p), L, n, n_pad, out.ctypes.data_as(C.c_void_p), cap,
                                    C.byref(nb))
    if st != QUEEN_OK:
        raise QueenError(st, f"queen_entropy_encode (needs {nb.value} bytes)")
    return out[: nb.value].copy()


def queen_set_sh_rest(ctx: Context, scene: QueenGaussians, latents, L: int, decoder, stream=None):
    """First-frame SH "set" decode: planes[14+m] = D . float(l) for the SH-rest rows."""
    st = lib().queen_set_sh_rest(ctx.handle, C.byref(scene), _ptr(latents), int(L), _ptr(decoder),
                                 C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_set_sh_rest")


def queen_entropy_decode(ctx: Context, stream_dev, L: int, n: int, latents_out, stream=None, nbytes: int | None = None):
    """stream_dev: device uint8 tensor holding one QANS stream (nbytes defaults to its size)."""
    nb = int(stream_dev.numel() * stream_dev.element_size()) if nbytes is None else int(nbytes)
    st = lib().queen_entropy_decode(ctx.handle, _ptr(stream_dev), nb, L, n, latents_out.shape[-1], _ptr(latents_out),
                                    C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_entropy_decode")


def queen_entropy_decode_frame(ctx: Context, stream_ptrs, stream_bytes, lat_dim, n: int, latents_out, stream=None):
    """Decode every category of a frame in one launch (stream_ptrs: 5 device addresses or None;
    stream_bytes: the 5 stream sizes)."""
    # (ctypes arrays are passed through: a caller decoding the same buffer every frame builds them once)
    ptrs = stream_ptrs if isinstance(stream_ptrs, C.Array) else \
        (C.c_void_p * 5)(*[C.c_void_p(int(p)) if p else None for p in stream_ptrs])
    nbs = stream_bytes if isinstance(stream_bytes, C.Array) else (C.c_int64 * 5)(*[int(x) for x in stream_bytes])
    dims = lat_dim if isinstance(lat_dim, C.Array) else (C.c_int32 * 5)(*[int(x) for x in lat_dim])
    st = lib().queen_entropy_decode_frame(ctx.handle, ptrs, nbs, dims, n, latents_out.shape[-1], _ptr(latents_out),
                                          C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_entropy_decode_frame")


def queen_wait_binned(ctx: Context, stream=None):
    st = lib().queen_wait_binned(ctx.handle, C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_wait_binned")


def queen_wait_projected(ctx: Context, stream=None):
    st = lib().queen_wait_projected(ctx.handle, C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_wait_projected")


def queen_set_blend_stream(ctx: Context, stream=None):
    """None: the blend runs on each render call's stream (default)."""
    st = lib().queen_set_blend_stream(ctx.handle, C.c_void_p(None if stream is None else stream.cuda_stream))
    ctx._chk(st, "queen_set_blend_stream")


def queen_wait_rendered(ctx: Context, stream=None):
    st = lib().queen_wait_rendered(ctx.handle, C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_wait_rendered")


def queen_blend_counts(ctx: Context, proj: QueenProj, bins: QueenBins, cams, evaluated, composited, stream=None):
    arr = camera_array(cams)
    st = lib().queen_blend_counts(ctx.handle, C.byref(proj), C.byref(bins), arr, len(cams), _ptr(evaluated),
                                  _ptr(composited), C.c_void_p(_stream(stream)))
    ctx._chk(st, "queen_blend_counts")
