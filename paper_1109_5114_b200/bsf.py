"""Thin Python binding of the C-ABI library ``libbsf.so`` (include/bsf.h).

Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  PyTorch provides device memory and streams.  There is no CPU
fallback: if the extension is missing, ``lib()`` raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BSF_LIB") or os.path.join(HERE, "libbsf.so")
LUT_DIR = os.path.join(HERE, "lut")

BSF_U8, BSF_F32, BSF_F64, BSF_I64, BSF_DD = 0, 1, 2, 3, 4
BSF_THETA, BSF_THETA_PRIME, BSF_DUAL = 0, 1, 2
BSF_PREC_FP64, BSF_PREC_DD, BSF_PREC_AUTO = 0, 1, 2
BSF_ANCHOR_GLOBAL, BSF_ANCHOR_TILE, BSF_ANCHOR_AUTO = 0, 1, 2

STATUS = {0: "ok", 1: "invalid argument", 2: "out of memory", 3: "CUDA error", 4: "infeasible covariance",
          5: "kernel reach exceeds plan margins", 6: "communication error", 7: "unsupported"}


class BsfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s (%d): %s" % (STATUS.get(status, "?"), status, msg))
        self.status = status


BSF_BOUNDARY_ZERO, BSF_BOUNDARY_REPLICATE = 0, 1
BSF_COV_SIGMA_THETA, BSF_COV_C11_C12_C22 = 0, 1


class bsf_plan_desc(ctypes.Structure):
    _fields_ = [("width", ctypes.c_int), ("height", ctypes.c_int), ("batch", ctypes.c_int),
                ("channels", ctypes.c_int), ("in_dtype", ctypes.c_int), ("out_dtype", ctypes.c_int),
                ("order", ctypes.c_int), ("basis", ctypes.c_int), ("max_sigma", ctypes.c_float),
                ("margin_x", ctypes.c_int), ("margin_y", ctypes.c_int), ("clamp", ctypes.c_int),
                ("precision", ctypes.c_int), ("device", ctypes.c_int), ("anchor", ctypes.c_int),
                ("boundary", ctypes.c_int), ("super_tile", ctypes.c_int), ("cov_layout", ctypes.c_int),
                ("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nccl_id", ctypes.c_void_p)]


class bsf_geometry(ctypes.Structure):
    _fields_ = [("margin_x", ctypes.c_int), ("margin_y", ctypes.c_int), ("g_width", ctypes.c_int),
                ("g_height", ctypes.c_int), ("nbases", ctypes.c_int), ("g_bytes", ctypes.c_size_t),
                ("g_exact_bytes", ctypes.c_size_t), ("super_tile", ctypes.c_int),
                ("global_mode", ctypes.c_int), ("tile_unit", ctypes.c_int), ("row0", ctypes.c_int),
                ("row_count", ctypes.c_int), ("block_row0", ctypes.c_int), ("block_rows", ctypes.c_int),
                ("halo", ctypes.c_int), ("g_row0", ctypes.c_int), ("g_rows", ctypes.c_int)]


class bsf_stats(ctypes.Structure):
    _fields_ = [("pixels", ctypes.c_longlong), ("clamped", ctypes.c_longlong), ("zero_scale", ctypes.c_longlong),
                ("theta_prime", ctypes.c_longlong), ("flags", ctypes.c_longlong),
                ("double_double", ctypes.c_longlong), ("macs", ctypes.c_longlong)]


_lib = None


def lib():
    """Load libbsf.so (built in-tree by build.py / __graft_entry__.build)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError("libbsf.so not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        vp, i, st = ctypes.c_void_p, ctypes.c_int, ctypes.c_int
        L.bsf_plan_create.restype = st
        L.bsf_plan_create.argtypes = [ctypes.POINTER(bsf_plan_desc), ctypes.c_char_p, ctypes.POINTER(vp)]
        L.bsf_plan_destroy.restype = st
        L.bsf_plan_destroy.argtypes = [vp]
        L.bsf_plan_geometry.restype = st
        L.bsf_plan_geometry.argtypes = [vp, ctypes.POINTER(bsf_geometry)]
        for name in ("bsf_preintegrate", "bsf_preintegrate_exact"):
            getattr(L, name).restype = st
            getattr(L, name).argtypes = [vp, vp, vp, vp]
        L.bsf_scan_step.restype = st
        L.bsf_scan_step.argtypes = [vp, i, i, ctypes.POINTER(i), ctypes.POINTER(i)]
        L.bsf_scan_level.restype = st
        L.bsf_scan_level.argtypes = [vp, i, i, i, vp, vp, vp, vp]
        L.bsf_filter_exact.restype = st
        L.bsf_filter_exact.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_filter.restype = st
        L.bsf_filter.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_filter_points.restype = st
        L.bsf_filter_points.argtypes = [vp, vp, vp, vp, i, vp, vp]
        L.bsf_filter_points_aux.restype = st
        L.bsf_filter_points_aux.argtypes = [vp, vp, vp, vp, i, vp, vp, vp]
        L.bsf_run_points.restype = st
        L.bsf_run_points.argtypes = [vp, vp, vp, vp, i, vp, vp, vp]
        L.bsf_run_tiles.restype = st
        L.bsf_run_tiles.argtypes = [vp, vp, vp, vp, vp, i, vp]
        L.bsf_run.restype = st
        L.bsf_run.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_run_normalized.restype = st
        L.bsf_run_normalized.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_run_alg1.restype = st
        L.bsf_run_alg1.argtypes = [vp, vp, vp, vp, vp, vp]
        L.bsf_run_split.restype = st
        L.bsf_run_split.argtypes = [vp, vp, vp, vp, i, ctypes.c_double, vp, vp]
        L.bsf_run_host.restype = st
        L.bsf_run_host.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_get_stats.restype = st
        L.bsf_get_stats.argtypes = [vp, ctypes.POINTER(bsf_stats), i]
        L.bsf_launch_count.restype = ctypes.c_longlong
        L.bsf_launch_count.argtypes = [vp]
        L.bsf_debug_phase_cycles.restype = st
        L.bsf_debug_phase_cycles.argtypes = [vp, vp, i]
        L.bsf_debug_item_cycles.restype = st
        L.bsf_debug_item_cycles.argtypes = [vp, vp, vp, i, vp, i]
        L.bsf_debug_option.restype = st
        L.bsf_debug_option.argtypes = [vp, ctypes.c_char_p, ctypes.c_double]
        L.bsf_uses_fused.restype = i
        L.bsf_uses_fused.argtypes = [vp]
        L.bsf_status_str.restype = ctypes.c_char_p
        L.bsf_status_str.argtypes = [st]
        L.bsf_last_error.restype = ctypes.c_char_p
        L.bsf_last_error.argtypes = []
        L.bsf_version.restype = i
        L.bsf_strip_rows.restype = st
        L.bsf_strip_rows.argtypes = [i, i, i, i, i] + [ctypes.POINTER(i)] * 4
        L.bsf_strip_exchange.restype = st
        L.bsf_strip_exchange.argtypes = [i, i, i, i, i, ctypes.POINTER(i)]
        L.bsf_get_unique_id.restype = st
        L.bsf_get_unique_id.argtypes = [vp]
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        raise BsfError(status, lib().bsf_last_error().decode())


def _stream(stream):
    if stream is None:
        import torch
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    return ctypes.c_void_p(t.data_ptr())


_IN_TORCH = {BSF_U8: "uint8", BSF_F32: "float32"}
_OUT_TORCH = {BSF_F64: "float64", BSF_F32: "float32"}


def _want(t, name, dtypes, numel, device=None):
    """Validate a tensor handed to the C ABI (which cannot check it): dtype,
    contiguity, element count and device (an int ordinal, or "cpu").  Raw
    integer pointers are passed through unchecked."""
    if t is None or isinstance(t, int):
        return
    dt = str(t.dtype).replace("torch.", "")
    if dt not in dtypes:
        raise BsfError(1, "%s: dtype %s, expected %s" % (name, dt, "/".join(dtypes)))
    if not t.is_contiguous():
        raise BsfError(1, "%s: not contiguous" % name)
    if t.numel() < numel:
        raise BsfError(1, "%s: %d elements, need %d" % (name, t.numel(), numel))
    if device == "cpu":
        if t.device.type != "cpu":
            raise BsfError(1, "%s: expected a host tensor" % name)
    elif device is not None and (t.device.type != "cuda" or t.device.index != device):
        raise BsfError(1, "%s: on %s, plan is on cuda:%d" % (name, t.device, device))


class Plan:
    """A bsf_plan_t.  Methods mirror the C functions of include/bsf.h."""

    def __init__(self, width, height, *, batch=1, channels=1, in_dtype=BSF_F32, out_dtype=BSF_F64, order=1,
                 basis=BSF_DUAL, max_sigma=1.0, margin_x=0, margin_y=0, clamp=1, precision=BSF_PREC_DD,
                 device=0, anchor=BSF_ANCHOR_GLOBAL, boundary=0, super_tile=0, cov_layout=BSF_COV_SIGMA_THETA,
                 rank=0, nranks=1, nccl_id=None, lut_dir=LUT_DIR):
        self._id = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        self.desc = bsf_plan_desc(width, height, batch, channels, in_dtype, out_dtype, order, basis,
                                  float(max_sigma), margin_x, margin_y, clamp, precision, device, anchor, boundary,
                                  super_tile, cov_layout, rank, nranks,
                                  ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None)
        h = ctypes.c_void_p()
        _check(lib().bsf_plan_create(ctypes.byref(self.desc), lut_dir.encode(), ctypes.byref(h)))
        self.handle = h
        g = bsf_geometry()
        _check(lib().bsf_plan_geometry(self.handle, ctypes.byref(g)))
        self.geometry = g

    def close(self):
        if getattr(self, "handle", None):
            lib().bsf_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # --- allocation helpers (PyTorch owns device memory) ---------------------
    def empty_g(self):
        import torch
        return torch.empty(self.geometry.g_bytes // 8, dtype=torch.float64, device="cuda:%d" % self.desc.device)

    def empty_g_exact(self):
        import torch
        n = self.geometry.g_exact_bytes // 8
        g = self.geometry
        return torch.empty(n, dtype=torch.int64, device="cuda:%d" % self.desc.device).view(
            g.nbases, self.desc.batch * self.desc.channels, g.g_height, g.g_width)

    # --- argument checks (the C ABI takes raw pointers) ------------------------
    def _rows(self):  # rows of cov / out (a row strip's own rows for multi-GPU plans)
        return self.geometry.row_count if self.desc.nranks > 1 else self.desc.height

    def _npix(self):
        d = self.desc
        return d.batch * d.channels * self._rows() * d.width

    def _check_f(self, f, device=None):
        d = self.desc
        rows = self._rows()
        if d.nranks > 1 and not d.nccl_id:
            rows = self.geometry.block_rows  # the caller assembled the block (own rows + halo)
        _want(f, "f", [_IN_TORCH[d.in_dtype]], d.batch * d.channels * rows * d.width,
              d.device if device is None else device)

    def _check_cov(self, cov, device=None):
        d = self.desc
        _want(cov, "cov", ["float32"], d.batch * 3 * self._rows() * d.width, d.device if device is None else device)

    def _check_out(self, out, device=None):
        _want(out, "out", [_OUT_TORCH[self.desc.out_dtype]], self._npix(),
              self.desc.device if device is None else device)

    # --- C-ABI calls ------------------------------------------------------------
    def preintegrate(self, f, g, stream=None):
        self._check_f(f)
        _want(g, "g", ["float64"], self.geometry.g_bytes // 8, self.desc.device)
        _check(lib().bsf_preintegrate(self.handle, _ptr(f), _ptr(g), _stream(stream)))

    def preintegrate_exact(self, f, g, stream=None):
        self._check_f(f)
        _want(g, "g", ["int64"], self.geometry.g_exact_bytes // 8, self.desc.device)
        _check(lib().bsf_preintegrate_exact(self.handle, _ptr(f), _ptr(g), _stream(stream)))

    def scan_step(self, slot, level):
        """(sx, sy) of running-sum level `level` of slot `slot`."""
        sx, sy = ctypes.c_int(), ctypes.c_int()
        _check(lib().bsf_scan_step(self.handle, slot, level, ctypes.byref(sx), ctypes.byref(sy)))
        return sx.value, sy.value

    def scan_level(self, slot, level, f, g, carry=None, exact=True, stream=None):
        """One pre-integration level in place on g (level 0 reads f); carry = the
        level's sums on the sy domain rows above this row strip, or None."""
        _check(lib().bsf_scan_level(self.handle, slot, level, 1 if exact else 0, _ptr(f), _ptr(g),
                                    _ptr(carry) if carry is not None else None, _stream(stream)))

    def filter(self, g, cov, out, stream=None):
        _want(g, "g", ["float64"], self.geometry.g_bytes // 8, self.desc.device)
        self._check_cov(cov)
        self._check_out(out)
        _check(lib().bsf_filter(self.handle, _ptr(g), _ptr(cov), _ptr(out), _stream(stream)))

    def filter_exact(self, g, cov, out, stream=None):
        """bsf_filter_exact: global-mode gather from bsf_preintegrate_exact's sums."""
        _want(g, "g", ["int64"], self.geometry.g_exact_bytes // 8, self.desc.device)
        self._check_cov(cov)
        self._check_out(out)
        _check(lib().bsf_filter_exact(self.handle, _ptr(g), _ptr(cov), _ptr(out), _stream(stream)))

    def _check_pts(self, pts, out, aux=None):
        n = pts.numel() // 3
        _want(pts, "pts", ["int32"], 3 * n, self.desc.device)
        _want(out, "out", ["float64"], n, self.desc.device)
        _want(aux, "aux", ["float64"], 12 * n, self.desc.device)
        return n

    def filter_points(self, g, cov, pts, out, stream=None):
        n = self._check_pts(pts, out)
        _want(cov, "cov", ["float32"], 3 * self.desc.height * self.desc.width, self.desc.device)
        _check(lib().bsf_filter_points(self.handle, _ptr(g), _ptr(cov), _ptr(pts), n, _ptr(out), _stream(stream)))

    def filter_points_aux(self, g, cov, pts, out, aux, stream=None):
        n = self._check_pts(pts, out, aux)
        _want(cov, "cov", ["float32"], 3 * self.desc.height * self.desc.width, self.desc.device)
        _check(lib().bsf_filter_points_aux(self.handle, _ptr(g), _ptr(cov), _ptr(pts), n, _ptr(out), _ptr(aux),
                                           _stream(stream)))

    def run_points(self, f, cov, pts, out, aux=None, stream=None):
        # points name their image: f and cov must hold every image the points
        # use (at least one; the caller guarantees the indices)
        n = self._check_pts(pts, out, aux)
        d = self.desc
        _want(f, "f", [_IN_TORCH[d.in_dtype]], d.height * d.width, d.device)
        _want(cov, "cov", ["float32"], 3 * d.height * d.width, d.device)
        _check(lib().bsf_run_points(self.handle, _ptr(f), _ptr(cov), _ptr(pts), n, _ptr(out), _ptr(aux),
                                    _stream(stream)))

    def run(self, f, cov, out, stream=None):
        self._check_f(f)
        self._check_cov(cov)
        self._check_out(out)
        _check(lib().bsf_run(self.handle, _ptr(f), _ptr(cov), _ptr(out), _stream(stream)))

    def run_tiles(self, f, cov, out, tiles, stream=None):
        """bsf_run_tiles: filter only the listed anchoring tiles (int32 indices)."""
        self._check_f(f)
        self._check_cov(cov)
        self._check_out(out)
        _want(tiles, "tiles", ["int32"], tiles.numel(), self.desc.device)
        _check(lib().bsf_run_tiles(self.handle, _ptr(f), _ptr(cov), _ptr(out), _ptr(tiles), int(tiles.numel()),
                                   _stream(stream)))

    def run_normalized(self, f, cov, out, stream=None):
        """DC-renormalised filter: out / filter(image indicator)."""
        self._check_f(f)
        self._check_cov(cov)
        self._check_out(out)
        _check(lib().bsf_run_normalized(self.handle, _ptr(f), _ptr(cov), _ptr(out), _stream(stream)))

    def run_alg1(self, f, cov, out, stream=None):
        """Algorithm 1 (covariance splitting); returns sigma_b^2 per covariance field."""
        import numpy as np
        self._check_f(f)
        self._check_cov(cov)
        self._check_out(out)
        sig = np.zeros(self.desc.batch, dtype=np.float64)
        _check(lib().bsf_run_alg1(self.handle, _ptr(f), _ptr(cov), _ptr(out),
                                  sig.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
        return sig

    def run_split(self, f, cov, out, passes, fraction=0.0, stream=None):
        """Generalised covariance splitting with `passes` passes and isotropic
        share `fraction` of the bound (0: (n-1)/n); returns sigma_b^2 per
        covariance field (the bound (9) is 2 sigma_b^2)."""
        import numpy as np
        self._check_f(f)
        self._check_cov(cov)
        self._check_out(out)
        sig = np.zeros(self.desc.batch, dtype=np.float64)
        _check(lib().bsf_run_split(self.handle, _ptr(f), _ptr(cov), _ptr(out), int(passes), float(fraction),
                                   sig.ctypes.data_as(ctypes.c_void_p), _stream(stream)))
        return sig

    def run_host(self, f_host, cov_host, out_host, stream=None):
        self._check_f(f_host, "cpu")
        self._check_cov(cov_host, "cpu")
        self._check_out(out_host, "cpu")
        _check(lib().bsf_run_host(self.handle, _ptr(f_host), _ptr(cov_host), _ptr(out_host), _stream(stream)))

    def stats(self, reset=False):
        s = bsf_stats()
        st = lib().bsf_get_stats(self.handle, ctypes.byref(s), 1 if reset else 0)
        d = {k: getattr(s, k) for k, _ in bsf_stats._fields_}
        d["status"] = st
        return d

    def phase_cycles(self, reset=False):
        """Per-phase SM cycles of the fused tile kernel (enables counting on first call)."""
        buf = (ctypes.c_ulonglong * 16)()
        _check(lib().bsf_debug_phase_cycles(self.handle, buf, int(reset)))
        return list(buf)

    def item_cycles(self, nitems, nctas=0):
        """(per-item cycles of the last run, per-item (MACs, fallback pixels,
        halo points, planes), per-CTA busy cycles since the last reset) of the
        fused tile kernel; phase_cycles() must have enabled the counters."""
        it = (ctypes.c_ulonglong * max(nitems, 1))()
        wk = (ctypes.c_ulonglong * max(4 * nitems, 1))()
        ct = (ctypes.c_ulonglong * max(nctas, 1))()
        _check(lib().bsf_debug_item_cycles(self.handle, it, wk, int(nitems), ct, int(nctas)))
        wl = list(wk)
        return list(it)[:nitems], [tuple(wl[4 * i:4 * i + 4]) for i in range(nitems)], list(ct)[:nctas]

    def debug_option(self, name, value):
        """Diagnostics options of bsf_debug_option (include/bsf.h)."""
        _check(lib().bsf_debug_option(self.handle, name.encode(), float(value)))

    def uses_fused(self):
        return bool(lib().bsf_uses_fused(self.handle))

    def launch_count(self):
        return lib().bsf_launch_count(self.handle)


def strip_rows(height, unit, halo, rank, nranks):
    """bsf_strip_rows: (y0, y1, b0, b1) of a row strip (pure host arithmetic)."""
    v = [ctypes.c_int() for _ in range(4)]
    _check(lib().bsf_strip_rows(int(height), int(unit), int(halo), int(rank), int(nranks), *[ctypes.byref(x) for x in v]))
    return tuple(x.value for x in v)


def strip_exchange(height, unit, halo, rank, nranks):
    """bsf_strip_exchange: the 8 row counts / offsets of a strip's halo exchange."""
    x = (ctypes.c_int * 8)()
    _check(lib().bsf_strip_exchange(int(height), int(unit), int(halo), int(rank), int(nranks), x))
    return list(x)


def get_unique_id() -> bytes:
    """bsf_get_unique_id: the 128-byte NCCL id (rank 0), to broadcast to all ranks."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().bsf_get_unique_id(buf))
    return buf.raw


# C-ABI names, re-exported (the binding keeps the library's vocabulary)
def bsf_plan_create(**kw):
    return Plan(**kw)


def bsf_preintegrate(plan, f, g, stream=None):
    plan.preintegrate(f, g, stream)


def bsf_preintegrate_exact(plan, f, g, stream=None):
    plan.preintegrate_exact(f, g, stream)


def bsf_filter(plan, g, cov, out, stream=None):
    plan.filter(g, cov, out, stream)


def bsf_filter_points(plan, g, cov, pts, out, stream=None):
    plan.filter_points(g, cov, pts, out, stream)


def bsf_run_points(plan, f, cov, pts, out, aux=None, stream=None):
    plan.run_points(f, cov, pts, out, aux, stream)


def bsf_run(plan, f, cov, out, stream=None):
    plan.run(f, cov, out, stream)


def bsf_run_host(plan, f_host, cov_host, out_host, stream=None):
    plan.run_host(f_host, cov_host, out_host, stream)


def bsf_get_stats(plan, reset=False):
    return plan.stats(reset)


def exported_symbols():
    """Function names declared in include/bsf.h."""
    import re
    hdr = os.path.join(os.path.dirname(HERE), "include", "bsf.h")
    src = open(hdr).read()
    return sorted(set(re.findall(r"\b(bsf_[a-z_]+)\s*\(", src)))
