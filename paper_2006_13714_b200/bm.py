"""Thin Python binding of include/sc_bm.h (argument marshalling only).

Every step of the path runs in libscbm.so's CUDA kernels; torch provides device memory,
the current stream and (in :mod:`.dist`) process groups. There is no CPU fallback: if the
library is missing or no sm_100 device is usable, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SCBM_LIB") or os.path.join(_HERE, "libscbm.so")  # SCBM_LIB: tuning builds

SC_DTYPE_U8, SC_DTYPE_F32 = 0, 1
SC_KERNEL_SIMT, SC_KERNEL_TC_I8, SC_KERNEL_SIMT_WARP, SC_KERNEL_BOX, SC_KERNEL_BOXF, SC_KERNEL_TC_F32 = 0, 1, 2, 3, 4, 5
STATUS = {0: "SC_OK", 1: "SC_ERR_INVALID_ARGUMENT", 2: "SC_ERR_UNSUPPORTED",
          3: "SC_ERR_OUT_OF_MEMORY", 4: "SC_ERR_CUDA", 5: "SC_ERR_WRONG_DEVICE", 6: "SC_ERR_OVERFLOW"}

SC_METRIC_L2, SC_METRIC_NCC = 0, 1
EXPORTED = ["sc_bm_plan", "sc_bm_plan_ex", "sc_bm_run", "sc_bm_run_batch", "sc_bm_run_rows", "sc_bm_run_host",
            "sc_bm_plan_info", "sc_bm_set_kernel", "sc_bm_destroy", "sc_status_string",
            "sc_bm_norm_map", "sc_bm_run_dense_debug", "sc_bm_set_timing", "sc_bm_get_timing", "sc_bm_group",
            "sc_bm_nlm_weights", "sc_bm_set_temporal", "sc_bm_debug_fix_count", "sc_bm_nlm_average",
            "sc_bm_run_temporal", "sc_bm_plan3d", "sc_bm_run3d", "sc_bm_set_packed", "sc_bm_packed_words",
            "sc_bm_unpack", "sc_bm_unpack_host"]


class ScError(RuntimeError):
    def __init__(self, fn, code):
        super().__init__(f"{fn} failed: {STATUS.get(code, code)}")
        self.code = code


class Info(ctypes.Structure):
    _fields_ = [("n_ref_y", ctypes.c_int64), ("n_ref_x", ctypes.c_int64), ("n_refs", ctypes.c_int64),
                ("min_candidates", ctypes.c_int64), ("max_candidates", ctypes.c_int64),
                ("total_candidates", ctypes.c_int64), ("workspace_bytes", ctypes.c_int64),
                ("frames_per_chunk", ctypes.c_int64), ("launches", ctypes.c_int64),
                ("kernel", ctypes.c_int32), ("device", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Timing(ctypes.Structure):
    _fields_ = [("norm_ms", ctypes.c_double), ("match_ms", ctypes.c_double),
                ("norm_chunks", ctypes.c_int64), ("match_launches", ctypes.c_int64)]


_lib = None


def load_library():
    """Load libscbm.so (built by ``python -m paper_2006_13714_b200.build``). Raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2006_13714_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    ci = ctypes.c_int
    L.sc_bm_plan.argtypes = [ci, ci, ci, ci, ci, ci, ci, ci, ctypes.POINTER(vp)]
    L.sc_bm_plan_ex.argtypes = [ci, ci, ci, ci, ci, ci, ci, ci, ci, ctypes.POINTER(vp)]
    L.sc_bm_run.argtypes = [vp, vp, vp, vp, vp]
    L.sc_bm_run_batch.argtypes = [vp, vp, i64, vp, vp, vp]
    L.sc_bm_run_rows.argtypes = [vp, vp, i64, i32, i32, vp, vp, vp]
    L.sc_bm_run_host.argtypes = [vp, vp, i64, vp, vp, vp]
    L.sc_bm_plan_info.argtypes = [vp, ctypes.POINTER(Info)]
    L.sc_bm_set_kernel.argtypes = [vp, i32]
    L.sc_bm_destroy.argtypes = [vp]
    L.sc_status_string.argtypes = [ci]
    L.sc_status_string.restype = ctypes.c_char_p
    L.sc_bm_norm_map.argtypes = [vp, vp, vp, vp]
    L.sc_bm_run_dense_debug.argtypes = [vp, vp, vp, vp]
    L.sc_bm_debug_fix_count.argtypes = [vp, ctypes.POINTER(i32)]
    L.sc_bm_nlm_average.argtypes = [vp, vp, ctypes.c_float, vp, vp]
    L.sc_bm_run_temporal.argtypes = [vp, vp, i64, i64, i64, i64, vp, vp, vp]
    L.sc_bm_set_timing.argtypes = [vp, i32]
    L.sc_bm_get_timing.argtypes = [vp, ctypes.POINTER(Timing)]
    L.sc_bm_group.argtypes = [vp, vp, i64, vp, vp, vp]
    L.sc_bm_nlm_weights.argtypes = [vp, vp, ctypes.c_float, vp, vp]
    L.sc_bm_set_temporal.argtypes = [vp, i32]
    L.sc_bm_plan3d.argtypes = [ci, ci, ci, ci, ci, ci, ci, ci, ci, ci, ctypes.POINTER(vp)]
    L.sc_bm_run3d.argtypes = [vp, vp, i64, vp, vp, vp]
    L.sc_bm_set_packed.argtypes = [vp, i64]
    L.sc_bm_packed_words.argtypes = [vp, i64, ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.sc_bm_unpack.argtypes = [vp, vp, i64, vp, vp, vp]
    L.sc_bm_unpack_host.argtypes = [ci, ci, ci, ci, ci, ci, vp, i64, vp, vp]
    for fn in EXPORTED:
        if fn != "sc_status_string":
            getattr(L, fn).restype = ci
    _lib = L
    return L


def _check(fn, code):
    if code != 0:
        raise ScError(fn, code)


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Plan:
    """A block-matching plan (``sc_bm_plan``) bound to the current CUDA device.

    dtype "u8" takes uint8 images and returns exact int32 distances; "f32" takes float32
    images and returns float32 distances. Images are [N, C, H, W] (or [C, H, W]) torch
    tensors on the plan's device, contiguous.
    """

    def __init__(self, H, W, C, b, stride, window, K, dtype="u8", metric="l2"):
        self._lib = load_library()
        self.H, self.W, self.C, self.b, self.s, self.Wn, self.K = H, W, C, b, stride, window, K
        self.dtype, self.metric = dtype, metric
        code = {"u8": SC_DTYPE_U8, "f32": SC_DTYPE_F32}[dtype]
        mcode = {"l2": SC_METRIC_L2, "ncc": SC_METRIC_NCC}[metric]
        h = ctypes.c_void_p()
        _check("sc_bm_plan_ex", self._lib.sc_bm_plan_ex(H, W, C, b, stride, window, K, code, mcode, ctypes.byref(h)))
        self._h = h
        inf = self.info()
        self.ny, self.nx, self.n_refs = inf["n_ref_y"], inf["n_ref_x"], inf["n_refs"]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.sc_bm_destroy(h)
            self._h = None

    close = __del__

    def info(self) -> dict:
        out = Info()
        _check("sc_bm_plan_info", self._lib.sc_bm_plan_info(self._h, ctypes.byref(out)))
        return out.as_dict()

    def set_timing(self, enable: bool):
        """Record per-kernel CUDA events on the run stream (bench roofline)."""
        _check("sc_bm_set_timing", self._lib.sc_bm_set_timing(self._h, int(enable)))

    def get_timing(self) -> dict:
        """Summed device ms of the norm / matching kernels since the last call (syncs on them)."""
        out = Timing()
        _check("sc_bm_get_timing", self._lib.sc_bm_get_timing(self._h, ctypes.byref(out)))
        return {k: getattr(out, k) for k, _ in out._fields_}

    def set_temporal(self, T: int):
        """Temporal search radius over the frames of a batch call (idx becomes batch-global)."""
        _check("sc_bm_set_temporal", self._lib.sc_bm_set_temporal(self._h, T))

    def set_kernel(self, kernel: int):
        _check("sc_bm_set_kernel", self._lib.sc_bm_set_kernel(self._h, kernel))

    def _dist_dtype(self):
        import torch
        return torch.int32 if (self.dtype == "u8" and self.metric == "l2") else torch.float32

    # ------------------------------------------------------------------ device paths
    def _check_img(self, imgs):
        import torch
        if imgs.dim() == 3:
            imgs = imgs.unsqueeze(0)
        want = torch.uint8 if self.dtype == "u8" else torch.float32
        if imgs.dtype != want or not imgs.is_cuda or not imgs.is_contiguous():
            raise ValueError(f"expected a contiguous CUDA {want} tensor [N,C,H,W]")
        if tuple(imgs.shape[1:]) != (self.C, self.H, self.W):
            raise ValueError(f"image shape {tuple(imgs.shape)} does not match the plan")
        return imgs

    def _check_out(self, out, n_images, refs, cuda):
        """Output tables must be contiguous [n, refs, K] int32 idx + dist of the plan's dtype,
        on the device (device paths) or in host memory (run_host): the C ABI writes
        n * refs * K elements through the raw pointers."""
        import torch
        idx, dist = out
        for name, t, want in (("idx", idx, torch.int32), ("dist", dist, self._dist_dtype())):
            if not isinstance(t, torch.Tensor) or t.dtype != want or t.is_cuda != cuda or \
                    not t.is_contiguous() or tuple(t.shape) != (n_images, refs, self.K):
                raise ValueError(f"{name} must be a contiguous {'CUDA' if cuda else 'host'} {want} tensor "
                                 f"of shape {(n_images, refs, self.K)}")
        return idx, dist

    def alloc_out(self, n_images, rows=None):
        import torch
        refs = self.n_refs if rows is None else (rows[1] - rows[0]) * self.nx
        dev = torch.device("cuda", torch.cuda.current_device())
        idx = torch.empty((n_images, refs, self.K), dtype=torch.int32, device=dev)
        dist = torch.empty((n_images, refs, self.K), dtype=self._dist_dtype(), device=dev)
        return idx, dist

    def run(self, imgs, out=None, stream=None):
        """Block matching on device tensors; returns (idx, dist) [N, n_refs, K]."""
        imgs = self._check_img(imgs)
        idx, dist = (self._check_out(out, imgs.shape[0], self.n_refs, True) if out is not None
                     else self.alloc_out(imgs.shape[0]))
        _check("sc_bm_run_batch", self._lib.sc_bm_run_batch(
            self._h, ctypes.c_void_p(imgs.data_ptr()), imgs.shape[0], ctypes.c_void_p(idx.data_ptr()),
            ctypes.c_void_p(dist.data_ptr()), _stream_ptr(stream)))
        return idx, dist

    def run_rows(self, imgs, iy_begin, iy_end, out=None, stream=None):
        """Only reference-grid rows [iy_begin, iy_end) (row-band sharding)."""
        imgs = self._check_img(imgs)
        if out is not None:
            out = self._check_out(out, imgs.shape[0], max(0, iy_end - iy_begin) * self.nx, True)
        idx, dist = out if out is not None else self.alloc_out(imgs.shape[0], (iy_begin, iy_end))
        _check("sc_bm_run_rows", self._lib.sc_bm_run_rows(
            self._h, ctypes.c_void_p(imgs.data_ptr()), imgs.shape[0], iy_begin, iy_end,
            ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()), _stream_ptr(stream)))
        return idx, dist

    def run_host(self, imgs: np.ndarray | "torch.Tensor", out=None, stream=None):
        """Host buffers in, host buffers out (pipelined H2D / match / D2H inside the library)."""
        import torch
        t = imgs if isinstance(imgs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(imgs))
        if t.dim() == 3:
            t = t.unsqueeze(0)
        want = torch.uint8 if self.dtype == "u8" else torch.float32
        if t.is_cuda or not t.is_contiguous() or t.dtype != want or t.dim() != 4 or \
                tuple(t.shape[1:]) != (self.C, self.H, self.W):
            raise ValueError(f"run_host expects a contiguous host {want} tensor/array [N, {self.C}, {self.H}, {self.W}]")
        n = t.shape[0]
        if out is None:
            idx = torch.empty((n, self.n_refs, self.K), dtype=torch.int32)
            dist = torch.empty((n, self.n_refs, self.K), dtype=self._dist_dtype())
        else:
            idx, dist = self._check_out(out, n, self.n_refs, False)
        _check("sc_bm_run_host", self._lib.sc_bm_run_host(
            self._h, ctypes.c_void_p(t.data_ptr()), n, ctypes.c_void_p(idx.data_ptr()),
            ctypes.c_void_p(dist.data_ptr()), _stream_ptr(stream)))
        return idx, dist

    # ------------------------------------------------------------------ packed tables (sc_bm_set_packed)
    def set_packed(self, cap_rows: int):
        """Packed tables: one uint32 word (dist << rb) | window slot per result, escape rows in an
        overflow area of cap_rows records (0: plain tables again)."""
        _check("sc_bm_set_packed", self._lib.sc_bm_set_packed(self._h, int(cap_rows)))

    def packed_words(self, n_images: int):
        """(words of a packed buffer for n_images images, slot bits rb)."""
        w, rb = ctypes.c_int64(0), ctypes.c_int32(0)
        _check("sc_bm_packed_words", self._lib.sc_bm_packed_words(self._h, int(n_images), ctypes.byref(w),
                                                                  ctypes.byref(rb)))
        return w.value, rb.value

    def _check_packed(self, buf, words, cuda):
        import torch
        if not isinstance(buf, torch.Tensor) or buf.dtype != torch.int32 or buf.is_cuda != cuda or \
                not buf.is_contiguous() or buf.numel() != words:
            raise ValueError(f"packed buffer must be a contiguous {'CUDA' if cuda else 'host'} int32 tensor "
                             f"of {words} words (uint32 bit patterns)")
        return buf

    def run_packed(self, imgs, out=None, stream=None):
        """Packed block matching on device tensors: an int32 tensor of packed_words(N) words."""
        import torch
        imgs = self._check_img(imgs)
        words, _ = self.packed_words(imgs.shape[0])
        buf = self._check_packed(out, words, True) if out is not None else \
            torch.empty(words, dtype=torch.int32, device=imgs.device)
        _check("sc_bm_run_batch", self._lib.sc_bm_run_batch(
            self._h, ctypes.c_void_p(imgs.data_ptr()), imgs.shape[0], ctypes.c_void_p(buf.data_ptr()),
            None, _stream_ptr(stream)))
        return buf

    def run_host_packed(self, imgs, out=None, stream=None):
        """Packed block matching, host buffers in and out (sc_bm_run_host in packed mode)."""
        import torch
        t = imgs if isinstance(imgs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(imgs))
        if t.dim() == 3:
            t = t.unsqueeze(0)
        if t.is_cuda or not t.is_contiguous() or t.dtype != torch.uint8 or t.dim() != 4 or \
                tuple(t.shape[1:]) != (self.C, self.H, self.W):
            raise ValueError(f"run_host_packed expects a contiguous host uint8 tensor/array [N, {self.C}, {self.H}, {self.W}]")
        words, _ = self.packed_words(t.shape[0])
        buf = self._check_packed(out, words, False) if out is not None else torch.empty(words, dtype=torch.int32)
        _check("sc_bm_run_host", self._lib.sc_bm_run_host(
            self._h, ctypes.c_void_p(t.data_ptr()), t.shape[0], ctypes.c_void_p(buf.data_ptr()), None,
            _stream_ptr(stream)))
        return buf

    def unpack(self, packed, n_images, out=None, stream=None):
        """Decode a device packed buffer of n_images images into the plain (idx, dist) tables."""
        words, _ = self.packed_words(n_images)
        packed = self._check_packed(packed, words, True)
        idx, dist = (self._check_out(out, n_images, self.n_refs, True) if out is not None
                     else self.alloc_out(n_images))
        _check("sc_bm_unpack", self._lib.sc_bm_unpack(
            self._h, ctypes.c_void_p(packed.data_ptr()), int(n_images), ctypes.c_void_p(idx.data_ptr()),
            ctypes.c_void_p(dist.data_ptr()), _stream_ptr(stream)))
        return idx, dist

    def group(self, imgs, idx, out=None, stream=None):
        """Patch groups Y_i of a run's idx table: [N, n_refs, K, C, b, b] (input dtype)."""
        import torch
        imgs = self._check_img(imgs)
        n = imgs.shape[0]
        if idx.dtype != torch.int32 or not idx.is_cuda or not idx.is_contiguous() or \
                tuple(idx.shape) != (n, self.n_refs, self.K):
            raise ValueError("idx must be the contiguous CUDA int32 [N, n_refs, K] table of a run")
        if out is None:
            out = torch.empty((n, self.n_refs, self.K, self.C, self.b, self.b), dtype=imgs.dtype, device=imgs.device)
        _check("sc_bm_group", self._lib.sc_bm_group(
            self._h, ctypes.c_void_p(imgs.data_ptr()), n, ctypes.c_void_p(idx.data_ptr()),
            ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def nlm_weights(self, img, h, out=None, stream=None):
        """NLM weights of one image [C,H,W] (or [1,C,H,W]): float32 [n_refs, Wn*Wn], rows sum to 1."""
        import torch
        img = self._check_img(img)[0]
        if out is None:
            out = torch.empty((self.n_refs, self.Wn * self.Wn), dtype=torch.float32, device=img.device)
        _check("sc_bm_nlm_weights", self._lib.sc_bm_nlm_weights(
            self._h, ctypes.c_void_p(img.data_ptr()), float(h), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    # ------------------------------------------------------------------ test exports
    def norm_map(self, img, stream=None):
        import torch
        img = self._check_img(img)[0]
        out = torch.empty((self.H - self.b + 1, self.W - self.b + 1),
                          dtype=torch.int32 if self.dtype == "u8" else torch.float32, device=img.device)
        _check("sc_bm_norm_map", self._lib.sc_bm_norm_map(
            self._h, ctypes.c_void_p(img.data_ptr()), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def dense_debug(self, img, stream=None):
        import torch
        img = self._check_img(img)[0]
        out = torch.empty((self.n_refs, self.Wn * self.Wn),
                          dtype=torch.int32 if self.dtype == "u8" else torch.float32, device=img.device)
        _check("sc_bm_run_dense_debug", self._lib.sc_bm_run_dense_debug(
            self._h, ctypes.c_void_p(img.data_ptr()), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def run_temporal(self, imgs, f_begin, f_end, frame_offset=0, out=None, stream=None):
        """Temporal search (set_temporal(T) first) for the reference frames [f_begin, f_end) of the
        batch imgs, candidates from every frame of it; idx = (frame + frame_offset) * H * W + pixel."""
        imgs = self._check_img(imgs)
        # (the C ABI validates the range: an empty allocation for an invalid one)
        idx, dist = out if out is not None else self.alloc_out(max(0, f_end - f_begin))
        _check("sc_bm_run_temporal", self._lib.sc_bm_run_temporal(
            self._h, ctypes.c_void_p(imgs.data_ptr()), imgs.shape[0], f_begin, f_end, frame_offset,
            ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()), _stream_ptr(stream)))
        return idx, dist

    def nlm_average(self, img, h, out=None, stream=None):
        """NL-means estimate of every reference patch (sum_j s_i(j) X_j), one image [C,H,W] (or
        [1,C,H,W]): float32 [n_refs, C, b, b]; the weights are never materialised."""
        import torch
        img = self._check_img(img)[0]
        if out is None:
            out = torch.empty((self.n_refs, self.C, self.b, self.b), dtype=torch.float32, device=img.device)
        _check("sc_bm_nlm_average", self._lib.sc_bm_nlm_average(
            self._h, ctypes.c_void_p(img.data_ptr()), float(h), ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def debug_fix_count(self):
        """References the last matching launch sent to the exact fix-up kernel (test export)."""
        n = ctypes.c_int32(0)
        _check("sc_bm_debug_fix_count", self._lib.sc_bm_debug_fix_count(self._h, ctypes.byref(n)))
        return n.value


class Plan3D(Plan):
    """3D block matching over the planes of a float volume (``sc_bm_plan3d`` / ``sc_bm_run3d``):
    patches of d planes x b x b, references every z_stride planes, candidates at z_window plane
    offsets x the clipped spatial window. ``run(vol [P,H,W])`` returns
    (idx, dist) [n_zref, n_refs, K], idx = (z * H + y) * W + x."""

    def __init__(self, H, W, d, b, stride, window, z_stride, z_window, K, dtype="f32"):
        self._lib = load_library()
        self.H, self.W, self.C, self.b, self.s, self.Wn, self.K = H, W, d, b, stride, window, K
        self.d, self.z_stride, self.z_window = d, z_stride, z_window
        self.dtype, self.metric = dtype, "l2"
        h = ctypes.c_void_p()
        _check("sc_bm_plan3d", self._lib.sc_bm_plan3d(H, W, d, b, stride, window, z_stride, z_window, K,
                                                      {"u8": SC_DTYPE_U8, "f32": SC_DTYPE_F32}[dtype], ctypes.byref(h)))
        self._h = h
        inf = self.info()
        self.ny, self.nx, self.n_refs = inf["n_ref_y"], inf["n_ref_x"], inf["n_refs"]

    def n_zref(self, n_planes: int) -> int:
        return (n_planes - self.d) // self.z_stride + 1

    def run(self, vol, out=None, stream=None):
        import torch
        v = vol.reshape(-1, self.H, self.W) if vol.dim() != 3 else vol
        if v.dtype != torch.float32 or not v.is_cuda or not v.is_contiguous():
            raise ValueError("expected a contiguous CUDA float32 volume [P, H, W]")
        nz = self.n_zref(v.shape[0])
        if out is None:
            idx, dist = self.alloc_out(nz)
        else:
            idx, dist = self._check_out(out, nz, self.n_refs, True)
        _check("sc_bm_run3d", self._lib.sc_bm_run3d(self._h, ctypes.c_void_p(v.data_ptr()), v.shape[0],
                                                    ctypes.c_void_p(idx.data_ptr()), ctypes.c_void_p(dist.data_ptr()),
                                                    _stream_ptr(stream)))
        return idx, dist


def unpack_host(H, W, b, stride, window, K, packed, n_images):
    """Host decode of a packed buffer (sc_bm_unpack_host; no device): numpy (idx, dist) int32
    [n_images, n_refs, K]. ``packed``: uint32/int32 numpy array (or host tensor) of the words."""
    L = load_library()
    p = np.ascontiguousarray(packed.numpy() if hasattr(packed, "numpy") else packed).view(np.uint32)
    ny, nx = (H - b) // stride + 1, (W - b) // stride + 1
    idx = np.empty((n_images, ny * nx, K), dtype=np.int32)
    dist = np.empty_like(idx)
    body = n_images * ny * nx * K
    if p.size < body + 2 or p.size < body + 2 + min(int(p[body]), int(p[body + 1])) * (2 + 2 * K):
        raise ValueError("packed buffer is shorter than its rows + overflow area")
    _check("sc_bm_unpack_host", L.sc_bm_unpack_host(H, W, b, stride, window, K, p.ctypes.data_as(ctypes.c_void_p),
                                                    int(n_images), idx.ctypes.data_as(ctypes.c_void_p),
                                                    dist.ctypes.data_as(ctypes.c_void_p)))
    return idx, dist


def status_string(code: int) -> str:
    return load_library().sc_status_string(code).decode()
