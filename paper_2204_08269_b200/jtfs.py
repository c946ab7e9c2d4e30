"""Thin ctypes binding of libjtfs.so (include/jtfs.h) -- argument marshalling only.

Every step of the JTFS path runs in the CUDA kernels behind the C ABI; this
module only converts Python / torch arguments to pointers and sizes.  There is
no CPU fallback: if the library is missing, importing the binding raises.

    plan = Plan(N=2**16, J=12, Q=16, J_fr=5, T=2**13, F=4)     # jtfs_plan_create
    out = plan.forward(x)       # x: torch.cuda.FloatTensor [B, N] -> [B, floats_per_signal]
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# JTFS_LIB: path of an alternative in-tree build (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("JTFS_LIB") or os.path.join(_HERE, "libjtfs.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2204_08269_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(LIB_PATH)

# --- status codes / constants (jtfs.h) ---
JTFS_OK, JTFS_ERR_INVALID_ARG, JTFS_ERR_UNSUPPORTED, JTFS_ERR_OOM = 0, 1, 2, 3
JTFS_ERR_CUDA, JTFS_ERR_WORKSPACE, JTFS_ERR_NONFINITE = 4, 5, 6
JTFS_CHECK_FINITE = 1
JTFS_LATENCY = 2
JTFS_KD_SIMT, JTFS_POOL_EXACT, JTFS_KD_PROF, JTFS_KD_NOPAIR = 4, 8, 16, 32  # validation / measurement plan flags
JTFS_PAD_REFLECT, JTFS_PAD_PERIODIC = 0, 1
PATH_SPIN, PATH_PSI_T_PHI_F, PATH_PHI_T_PSI_F, PATH_PHI_T_PHI_F = 0, 1, 2, 3

EXPORTS = [
    "jtfs_plan", "jtfs_plan_create", "jtfs_plan_destroy", "jtfs_layout", "jtfs_paths",
    "jtfs_lambda_xi", "jtfs_workspace_size", "jtfs_forward", "jtfs_forward_host",
    "jtfs_debug_tap", "jtfs_debug_tap_size", "jtfs_debug_filter", "jtfs_debug_joint", "jtfs_debug_fft",
    "jtfs_debug_a16_density", "jtfs_debug_kd_tiling",
    "jtfs_measure_fp32_peak", "jtfs_cost", "jtfs_profile_enable",
    "jtfs_profile_read", "jtfs_profile_read_kd", "jtfs_status_string", "jtfs_last_error",
    "jtfs_units", "jtfs_partials_size", "jtfs_forward_units", "jtfs_reduce_pack",
    "jtfs_unitset_create", "jtfs_unitset_destroy", "jtfs_forward_unitset", "jtfs_unit_partials_range",
    "jtfs_scat1d_layout", "jtfs_scat1d_paths", "jtfs_scattering1d",
    "jtfs_backward_workspace_size", "jtfs_backward", "jtfs_backward_regions", "jtfs_resynth_loss",
    "jtfs_mulog_mu", "jtfs_mulog_apply", "jtfs_forward_mulog", "jtfs_u2_map_shape", "jtfs_u2_map",
    "jtfs_knn_workspace_size", "jtfs_knn_regress", "jtfs_isomap_workspace_size", "jtfs_isomap",
]
STAGES = ["KA_pad_fft", "KB_first_order", "KS_phi_avg", "KC_second_order", "KD_joint", "KE_pool_pack"]


class jtfs_params(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("N", "J", "Q", "Q2", "T", "J_fr", "Q_fr", "F", "average_fr", "pad_mode", "device")] + \
               [("flags", C.c_uint32)]


class jtfs_layout_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("n1", "n_frames", "frame0", "lambda_out", "n_paths", "n_alpha", "n_beta", "N_pad",
                 "N_fr", "reserved")] + \
               [(n, C.c_int64) for n in ("off_s0", "off_s1", "off_s2", "floats_per_signal")]


class jtfs_path_t(C.Structure):
    _fields_ = [("kind", C.c_int32), ("theta", C.c_int32), ("alpha", C.c_int32), ("beta", C.c_int32),
                ("xi_alpha", C.c_double), ("xi_beta", C.c_double)]


class jtfs_scat1d_layout_t(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n1", "n2", "n_frames", "frame0")] + \
               [(n, C.c_int64) for n in ("off_s0", "off_s1", "off_s2", "floats_per_signal")]


class jtfs_unit_t(C.Structure):
    _fields_ = [("alpha", C.c_int32), ("chunk", C.c_int32), ("col0", C.c_int32), ("ncols", C.c_int32),
                ("cost", C.c_double)]


_P = C.c_void_p
_lib.jtfs_plan.argtypes = [C.c_int] * 8 + [C.POINTER(_P)]
_lib.jtfs_plan_create.argtypes = [C.POINTER(jtfs_params), C.POINTER(_P)]
_lib.jtfs_plan_destroy.argtypes = [_P]
_lib.jtfs_layout.argtypes = [_P, C.POINTER(jtfs_layout_t)]
_lib.jtfs_paths.argtypes = [_P, C.POINTER(jtfs_path_t), C.c_int32]
_lib.jtfs_lambda_xi.argtypes = [_P, C.POINTER(C.c_double), C.c_int32]
_lib.jtfs_workspace_size.argtypes = [_P, C.c_int64, C.POINTER(C.c_size_t)]
_lib.jtfs_forward.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_size_t, _P]
_lib.jtfs_forward_host.argtypes = [_P, _P, C.c_int64, _P, _P, _P, _P, C.c_size_t, _P]
_lib.jtfs_debug_tap.argtypes = [_P, C.c_int32, _P, C.c_int64, _P, C.c_int64, _P, C.c_size_t, _P]
_lib.jtfs_debug_tap_size.argtypes = [_P, C.c_int32, C.c_int64, C.POINTER(C.c_int64)]
_lib.jtfs_debug_joint.argtypes = [_P, _P, _P, C.c_int64, _P, _P, C.c_size_t, _P]
_lib.jtfs_debug_fft.argtypes = [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, C.c_int64, _P, C.c_size_t, _P]
_lib.jtfs_debug_a16_density.argtypes = [_P, C.c_double, C.POINTER(C.c_int64), C.c_int32]
_lib.jtfs_debug_kd_tiling.argtypes = [_P, C.POINTER(C.c_int32), C.c_int32]
KD_TILING_FIELDS = ("kd_impl", "pair", "stat", "Nt", "mpart", "mblk", "NBB", "S", "nkc", "pool_mode")
_lib.jtfs_measure_fp32_peak.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]
_lib.jtfs_debug_filter.argtypes = [_P, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
_lib.jtfs_cost.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32]
_lib.jtfs_profile_enable.argtypes = [_P, C.c_int32]
_lib.jtfs_profile_read.argtypes = [_P, C.POINTER(C.c_double), C.POINTER(C.c_int64), C.c_int32, C.c_int32]
_lib.jtfs_profile_read_kd.argtypes = [_P, C.POINTER(C.c_double), C.c_int32, C.c_int32]
_lib.jtfs_units.argtypes = [_P, C.POINTER(jtfs_unit_t), C.c_int32, C.POINTER(C.c_int32)]
_lib.jtfs_partials_size.argtypes = [_P, C.POINTER(C.c_int64)]
_lib.jtfs_forward_units.argtypes = [_P, _P, C.c_int64, C.POINTER(C.c_int32), C.c_int32, _P, _P, _P, C.c_size_t, _P]
_lib.jtfs_unitset_create.argtypes = [_P, C.POINTER(C.c_int32), C.c_int32, C.POINTER(_P)]
_lib.jtfs_unitset_destroy.argtypes = [_P]
_lib.jtfs_forward_unitset.argtypes = [_P, _P, C.c_int64, _P, _P, _P, _P, C.c_size_t, _P]
_lib.jtfs_unit_partials_range.argtypes = [_P, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
_lib.jtfs_reduce_pack.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_size_t, _P]
_lib.jtfs_scat1d_layout.argtypes = [_P, C.POINTER(jtfs_scat1d_layout_t)]
_lib.jtfs_scat1d_paths.argtypes = [_P, C.POINTER(C.c_int32), C.c_int32]
_lib.jtfs_scattering1d.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_size_t, _P]
_lib.jtfs_backward_workspace_size.argtypes = [_P, C.c_int64, C.POINTER(C.c_size_t)]
_lib.jtfs_backward.argtypes = [_P, _P, C.c_int64, _P, _P, _P, C.c_size_t, _P]
_lib.jtfs_resynth_loss.argtypes = [_P, _P, _P, _P, _P, _P]
_lib.jtfs_backward_regions.argtypes = [_P, C.c_int64, C.POINTER(C.c_int64), C.c_int32]
_lib.jtfs_mulog_mu.argtypes = [_P, _P, C.c_int64, _P, _P]
_lib.jtfs_mulog_apply.argtypes = [_P, _P, C.c_int64, _P, C.c_float, _P, _P]
_lib.jtfs_forward_mulog.argtypes = [_P, _P, C.c_int64, _P, C.c_float, _P, _P, C.c_size_t, _P]
_lib.jtfs_u2_map_shape.argtypes = [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
_lib.jtfs_u2_map.argtypes = [_P, _P, C.c_int64, C.c_int32, _P, _P, C.c_size_t, _P]
_lib.jtfs_knn_workspace_size.argtypes = [C.c_int64, C.POINTER(C.c_size_t)]
_lib.jtfs_knn_regress.argtypes = [_P, C.c_int64, C.c_int64, C.c_int64, _P, C.c_int32, C.c_int32, _P, _P, _P, _P,
                                  C.c_size_t, _P]
_lib.jtfs_isomap_workspace_size.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_size_t)]
_lib.jtfs_isomap.argtypes = [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, C.c_size_t, _P]
_lib.jtfs_status_string.argtypes = [C.c_int]
_lib.jtfs_status_string.restype = C.c_char_p
_lib.jtfs_last_error.argtypes = []
_lib.jtfs_last_error.restype = C.c_char_p
for _n in EXPORTS:
    if _n not in ("jtfs_status_string", "jtfs_last_error"):
        getattr(_lib, _n).restype = C.c_int


class JTFSError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = _lib.jtfs_last_error().decode(errors="replace")
        super().__init__(f"{where}: {_lib.jtfs_status_string(status).decode()} ({status}): {msg}")


def _check(status: int, where: str) -> None:
    if status != JTFS_OK:
        raise JTFSError(status, where)


def library():
    """The loaded ctypes CDLL (for symbol checks)."""
    return _lib


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def _stream_handle(stream) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream().cuda_stream)
    return int(getattr(stream, "cuda_stream", stream))


class Plan:
    """jtfs_plan_create / jtfs_plan_destroy and the queries of jtfs.h."""

    def __init__(self, N: int, J: int, Q: int, J_fr: int, T: int, F: int = 0, Q2: int = 1,
                 Q_fr: int = 1, average_fr: bool = True, pad_mode: int = JTFS_PAD_REFLECT,
                 device: int | None = None, flags: int = 0):
        if device is None:
            import torch
            device = torch.cuda.current_device() if torch.cuda.is_available() else -1
        self.params = jtfs_params(N, J, Q, Q2, T, J_fr, Q_fr, F, int(bool(average_fr)), pad_mode,
                                  device, flags)
        h = _P()
        _check(_lib.jtfs_plan_create(C.byref(self.params), C.byref(h)), "jtfs_plan_create")
        self._h = h
        lay = jtfs_layout_t()
        _check(_lib.jtfs_layout(self._h, C.byref(lay)), "jtfs_layout")
        self.layout = lay
        self.device = device
        self._ws = None

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            _lib.jtfs_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- queries ----
    @property
    def floats_per_signal(self) -> int:
        return int(self.layout.floats_per_signal)

    def paths(self):
        n = self.layout.n_paths
        arr = (jtfs_path_t * n)()
        _check(_lib.jtfs_paths(self._h, arr, n), "jtfs_paths")
        return [(p.kind, p.theta, p.alpha, p.beta, p.xi_alpha, p.xi_beta) for p in arr]

    def lambda_xi(self):
        n = self.layout.n1
        arr = (C.c_double * n)()
        _check(_lib.jtfs_lambda_xi(self._h, arr, n), "jtfs_lambda_xi")
        return list(arr)

    def workspace_size(self, batch: int) -> int:
        v = C.c_size_t()
        _check(_lib.jtfs_workspace_size(self._h, batch, C.byref(v)), "jtfs_workspace_size")
        return int(v.value)

    def debug_filter(self, bank: int, idx: int, L: int, n_grid: int):
        arr = (C.c_double * L)()
        _check(_lib.jtfs_debug_filter(self._h, bank, idx, L, n_grid, arr), "jtfs_debug_filter")
        return list(arr)

    def cost(self):
        """{stage: (algorithmic flops, bytes)} per signal (jtfs_cost)."""
        f = (C.c_double * 7)()
        b = (C.c_double * 7)()
        _check(_lib.jtfs_cost(self._h, f, b, 7), "jtfs_cost")
        out = {STAGES[i]: (f[i], b[i]) for i in range(6)}
        out["KD_tensor_executed"] = (f[6], b[6])
        return out

    # ---- tracing ----
    def profile_enable(self, on: bool = True):
        _check(_lib.jtfs_profile_enable(self._h, int(on)), "jtfs_profile_enable")

    def profile_read(self, reset: bool = True):
        """{stage: (ms, launches)} since the last reset (synchronises on the events)."""
        ms = (C.c_double * 6)()
        nl = (C.c_int64 * 6)()
        _check(_lib.jtfs_profile_read(self._h, ms, nl, 6, int(reset)), "jtfs_profile_read")
        return {STAGES[i]: (ms[i], nl[i]) for i in range(6)}

    def profile_read_kd(self, reset: bool = True):
        """Per-alpha KD milliseconds since the last reset."""
        n = self.layout.n_alpha
        ms = (C.c_double * max(n, 1))()
        _check(_lib.jtfs_profile_read_kd(self._h, ms, n, int(reset)), "jtfs_profile_read_kd")
        return [ms[i] for i in range(n)]

    # ---- compute (torch tensors on the plan's device) ----
    def workspace(self, batch: int, stream=None):
        """The cached workspace of `stream` (one per stream: forwards on different streams
        never share buffers; a buffer that grows is released only through the caching
        allocator's stream-ordered free, on the stream that used it)."""
        import torch
        need = self.workspace_size(batch)
        key = _stream_handle(stream)
        if self._ws is None:
            self._ws = {}
        ws = self._ws.get(key)
        if ws is None or ws.numel() < need:
            if ws is not None and stream is not None:
                ws.record_stream(stream if isinstance(stream, torch.cuda.Stream) else torch.cuda.current_stream())
            ws = torch.empty(need, dtype=torch.uint8, device=f"cuda:{self.device}")
            self._ws[key] = ws
        return ws

    def forward(self, x, out=None, stream=None):
        """x: float32 CUDA tensor [B, N] (contiguous) -> out [B, floats_per_signal]."""
        import torch
        assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous() and x.dim() == 2
        B = x.shape[0]
        if out is None:
            out = torch.empty(B, self.floats_per_signal, dtype=torch.float32, device=x.device)
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_forward(self._h, _ptr(x), B, _ptr(out), _ptr(ws), ws.numel(),
                                 _stream_handle(stream)), "jtfs_forward")
        return out

    def forward_host(self, x_host, out_host, x_dev, out_dev, stream=None):
        """End to end through the C ABI with HOST buffers (pinned torch CPU tensors)."""
        B = x_host.shape[0]
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_forward_host(self._h, _ptr(x_host), B, _ptr(out_host), _ptr(x_dev), _ptr(out_dev),
                                      _ptr(ws), ws.numel(), _stream_handle(stream)), "jtfs_forward_host")
        return out_host

    # ---- path sharding (jtfs_units / jtfs_forward_units / jtfs_reduce_pack) ----
    def units(self):
        """KD work units of one signal: list of dicts (alpha, chunk, col0, ncols, cost); id = index."""
        n = C.c_int32()
        _check(_lib.jtfs_units(self._h, None, 0, C.byref(n)), "jtfs_units")
        arr = (jtfs_unit_t * max(n.value, 1))()
        _check(_lib.jtfs_units(self._h, arr, n.value, C.byref(n)), "jtfs_units")
        return [dict(alpha=u.alpha, chunk=u.chunk, col0=u.col0, ncols=u.ncols, cost=u.cost)
                for u in arr[:n.value]]

    @property
    def partials_size(self) -> int:
        v = C.c_int64()
        _check(_lib.jtfs_partials_size(self._h, C.byref(v)), "jtfs_partials_size")
        return int(v.value)

    def forward_units(self, x, unit_ids, partials, out, stream=None):
        """KA..KC + S0/S1 into out + KD partials of the listed units (others zeroed)."""
        B = x.shape[0]
        ids = (C.c_int32 * max(len(unit_ids), 1))(*[int(i) for i in unit_ids])
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_forward_units(self._h, _ptr(x), B, ids, len(unit_ids), _ptr(partials), _ptr(out),
                                       _ptr(ws), ws.numel(), _stream_handle(stream)), "jtfs_forward_units")
        return partials, out

    def unitset(self, unit_ids):
        """A unit set bound to device tables once (jtfs_unitset_create)."""
        return UnitSet(self, unit_ids)

    def forward_unitset(self, x, uset, partials, out, stream=None):
        """forward_units with a bound set: asynchronous, graph-capturable (jtfs_forward_unitset)."""
        B = x.shape[0]
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_forward_unitset(self._h, _ptr(x), B, uset.handle, _ptr(partials), _ptr(out), _ptr(ws),
                                         ws.numel(), _stream_handle(stream)), "jtfs_forward_unitset")
        return partials, out

    def unit_partials_range(self, unit: int):
        """[begin, end) floats of one signal's partials that unit `unit` writes."""
        a, b = C.c_int64(), C.c_int64()
        _check(_lib.jtfs_unit_partials_range(self._h, unit, C.byref(a), C.byref(b)), "jtfs_unit_partials_range")
        return a.value, b.value

    def reduce_pack(self, partials, out, stream=None):
        """phi_F pooling + phi paths + packing of S2 from summed partials (same workspace)."""
        B = partials.shape[0]
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_reduce_pack(self._h, _ptr(partials), B, _ptr(out), _ptr(ws), ws.numel(),
                                     _stream_handle(stream)), "jtfs_reduce_pack")
        return out

    # ---- backward (vector-Jacobian product; jtfs_backward) ----
    def backward(self, x, dout, dx=None, stream=None):
        """dx = d<dout, forward(x)>/dx (x float32 CUDA [B, N], dout [B, floats_per_signal])."""
        import torch
        assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous() and dout.is_contiguous()
        B = x.shape[0]
        if dx is None:
            dx = torch.empty_like(x)
        n = C.c_size_t()
        _check(_lib.jtfs_backward_workspace_size(self._h, B, C.byref(n)), "jtfs_backward_workspace_size")
        if getattr(self, "_bws", None) is None or self._bws.numel() < n.value:
            self._bws = torch.empty(max(n.value, 1), dtype=torch.uint8, device=x.device)
        _check(_lib.jtfs_backward(self._h, _ptr(x), B, _ptr(dout), _ptr(dx), _ptr(self._bws), self._bws.numel(),
                                  _stream_handle(stream)), "jtfs_backward")
        return dx

    def resynth_loss(self, Sy, Sx, stream=None):
        """(E as a device fp64 scalar tensor, dE/dSy) for one record (jtfs_resynth_loss)."""
        import torch
        assert Sy.is_contiguous() and Sx.is_contiguous() and Sy.numel() == Sx.numel() == self.floats_per_signal
        E = torch.empty((), dtype=torch.float64, device=Sy.device)
        dout = torch.empty_like(Sy)
        _check(_lib.jtfs_resynth_loss(self._h, _ptr(Sy), _ptr(Sx), _ptr(E), _ptr(dout), _stream_handle(stream)),
               "jtfs_resynth_loss")
        return E, dout

    def backward_regions(self, B: int):
        """Byte offsets of the backward workspace regions (jtfs_backward_regions)."""
        arr = (C.c_int64 * 18)()
        _check(_lib.jtfs_backward_regions(self._h, B, arr, 18), "jtfs_backward_regions")
        return list(arr)

    # ---- second-order time scattering (jtfs_scat1d_layout / _paths / jtfs_scattering1d) ----
    @property
    def scat1d_layout(self):
        lay = jtfs_scat1d_layout_t()
        _check(_lib.jtfs_scat1d_layout(self._h, C.byref(lay)), "jtfs_scat1d_layout")
        return lay

    def scat1d_paths(self):
        """[(lambda, alpha)] of every S2_t row."""
        n = self.scat1d_layout.n2
        arr = (C.c_int32 * max(2 * n, 1))()
        _check(_lib.jtfs_scat1d_paths(self._h, arr, n), "jtfs_scat1d_paths")
        return [(arr[2 * r], arr[2 * r + 1]) for r in range(n)]

    def scattering1d(self, x, out=None, stream=None):
        """Time scattering: x float32 CUDA [B, N] -> [B, n_frames (1 + n1 + n2)]."""
        import torch
        assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous() and x.dim() == 2
        B = x.shape[0]
        lay = self.scat1d_layout
        if out is None:
            out = torch.empty(B, lay.floats_per_signal, dtype=torch.float32, device=x.device)
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_scattering1d(self._h, _ptr(x), B, _ptr(out), _ptr(ws), ws.numel(),
                                      _stream_handle(stream)), "jtfs_scattering1d")
        return out

    def unpack_scat1d(self, out):
        lay = self.scat1d_layout
        fr = lay.n_frames
        return (out[..., lay.off_s0:lay.off_s0 + fr],
                out[..., lay.off_s1:lay.off_s2].reshape(*out.shape[:-1], lay.n1, fr),
                out[..., lay.off_s2:].reshape(*out.shape[:-1], lay.n2, fr))

    def debug_tap(self, tap: int, x, stream=None):
        import torch
        B = x.shape[0]
        n = C.c_int64()
        _check(_lib.jtfs_debug_tap_size(self._h, tap, B, C.byref(n)), "jtfs_debug_tap_size")
        out = torch.empty(int(n.value), dtype=torch.float32, device=x.device)
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_debug_tap(self._h, tap, _ptr(x), B, _ptr(out), out.numel(), _ptr(ws), ws.numel(),
                                   _stream_handle(stream)), "jtfs_debug_tap")
        return out

    def debug_joint(self, y2, yphi, out=None, stream=None):
        """Joint stage (KD + KE) from given Y2 (tap-2 layout, float32 CUDA [B, 2 y2_total])
        and Y_phi (tap-3 layout, [B, n1 * N_pad/T]) -> out [B, floats_per_signal]."""
        import torch
        assert y2.dtype == torch.float32 and y2.is_cuda and y2.is_contiguous() and y2.dim() == 2
        assert yphi.dtype == torch.float32 and yphi.is_cuda and yphi.is_contiguous()
        B = y2.shape[0]
        if out is None:
            out = torch.empty(B, self.floats_per_signal, dtype=torch.float32, device=y2.device)
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_debug_joint(self._h, _ptr(y2), _ptr(yphi), B, _ptr(out), _ptr(ws), ws.numel(),
                                     _stream_handle(stream)), "jtfs_debug_joint")
        return out

    def kd_tiling(self):
        """Per alpha, the KD tiling the plan chose (dict of KD_TILING_FIELDS)."""
        n = self.layout.n_alpha
        out = (C.c_int32 * (10 * n))()
        _check(_lib.jtfs_debug_kd_tiling(self._h, out, 10 * n), "jtfs_debug_kd_tiling")
        return [dict(zip(KD_TILING_FIELDS, out[10 * i:10 * i + 10])) for i in range(n)]

    def a16_density(self, thr: float):
        """Per alpha (records, records with an entry > thr x row max, records in the per-block
        band, K-chunks per block, coefficients > thr x row max, coefficients) of the KD's tensor-core
        operand (host tables only)."""
        n = self.layout.n_alpha
        out = (C.c_int64 * (6 * n))()
        _check(_lib.jtfs_debug_a16_density(self._h, thr, out, 6 * n), "jtfs_debug_a16_density")
        return [tuple(out[6 * i:6 * i + 6]) for i in range(n)]

    def debug_fft(self, x, dir: int = -1, stream=None):
        """The FFT engine on rows of x (complex64 -> fp32 engine, complex128 -> fp64 engine)."""
        import torch
        assert x.is_cuda and x.is_contiguous() and x.dim() == 2 and x.dtype in (torch.complex64, torch.complex128)
        rows, L = x.shape
        lg = L.bit_length() - 1
        out = torch.empty_like(x)
        tmp = torch.empty_like(x)
        _check(_lib.jtfs_debug_fft(self._h, lg, dir, int(x.dtype == torch.complex128), _ptr(x), _ptr(out), rows,
                                   _ptr(tmp), tmp.numel() * tmp.element_size(), _stream_handle(stream)),
               "jtfs_debug_fft")
        return out

    # ---- NEXT-4: mu-log (Eqs. (adalog:mu), (adalog)) and the Fig. 1 map ----
    def mulog_mu(self, S, stream=None):
        """mu(lambda_2) of a batch of records S [B, floats_per_signal] -> float32 CUDA [n_paths]."""
        import torch
        assert S.dtype == torch.float32 and S.is_cuda and S.is_contiguous() and S.dim() == 2
        mu = torch.empty(self.layout.n_paths, dtype=torch.float32, device=S.device)
        _check(_lib.jtfs_mulog_mu(self._h, _ptr(S), S.shape[0], _ptr(mu), _stream_handle(stream)),
               "jtfs_mulog_mu")
        return mu

    def mulog_apply(self, S, mu, eps: float = 0.1, out=None, stream=None):
        """Records with every S2 value replaced by log(1 + S / (eps mu)); S0/S1 unchanged."""
        import torch
        assert S.dtype == torch.float32 and S.is_cuda and S.is_contiguous() and S.dim() == 2
        if out is None:
            out = torch.empty_like(S)
        _check(_lib.jtfs_mulog_apply(self._h, _ptr(S), S.shape[0], _ptr(mu), float(eps), _ptr(out),
                                     _stream_handle(stream)), "jtfs_mulog_apply")
        return out

    def forward_mulog(self, x, mu, eps: float = 0.1, out=None, stream=None):
        """jtfs_forward with the mu-log fused into KE."""
        import torch
        assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous() and x.dim() == 2
        B = x.shape[0]
        if out is None:
            out = torch.empty(B, self.floats_per_signal, dtype=torch.float32, device=x.device)
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_forward_mulog(self._h, _ptr(x), B, _ptr(mu), float(eps), _ptr(out), _ptr(ws),
                                       ws.numel(), _stream_handle(stream)), "jtfs_forward_mulog")
        return out

    def u2_map_shape(self, path: int):
        r, c = C.c_int32(), C.c_int32()
        _check(_lib.jtfs_u2_map_shape(self._h, path, C.byref(r), C.byref(c)), "jtfs_u2_map_shape")
        return r.value, c.value

    def u2_map(self, x, path: int, out=None, stream=None):
        """Scale-rate map |X * Psi| of S2 path `path` before Phi: x [B, N] -> [B, rows, cols]."""
        import torch
        assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous() and x.dim() == 2
        rows, cols = self.u2_map_shape(path)
        B = x.shape[0]
        if out is None:
            out = torch.empty(B, rows, cols, dtype=torch.float32, device=x.device)
        ws = self.workspace(B, stream)
        _check(_lib.jtfs_u2_map(self._h, _ptr(x), B, path, _ptr(out), _ptr(ws), ws.numel(),
                                _stream_handle(stream)), "jtfs_u2_map")
        return out

    # ---- unpack the out_3D record ----
    def unpack(self, out):
        L = self.layout
        fr = L.n_frames
        s0 = out[..., L.off_s0:L.off_s0 + fr]
        s1 = out[..., L.off_s1:L.off_s2].reshape(*out.shape[:-1], L.n1, fr)
        s2 = out[..., L.off_s2:].reshape(*out.shape[:-1], L.n_paths, L.lambda_out, fr)
        return s0, s1, s2


def knn_regress(F, theta=None, K: int = 40, stream=None):
    """K-NN parameter regression of feature rows F (float32 CUDA [n, d], row
    stride may exceed d) with parameters theta (float64 CUDA [n, P] or None).
    Returns (nbr int32 [n, K], theta_hat float64 [n, P] | None, ratio float64 [n, P] | None)."""
    import torch
    assert F.dtype == torch.float32 and F.is_cuda and F.dim() == 2 and F.stride(1) == 1
    n, d = F.shape
    P = 0 if theta is None else theta.shape[1]
    if theta is not None:
        assert theta.dtype == torch.float64 and theta.is_cuda and theta.is_contiguous() and theta.shape[0] == n
    sz = C.c_size_t()
    _check(_lib.jtfs_knn_workspace_size(n, C.byref(sz)), "jtfs_knn_workspace_size")
    ws = torch.empty(max(int(sz.value), 1), dtype=torch.uint8, device=F.device)
    nbr = torch.empty(n, K, dtype=torch.int32, device=F.device)
    hat = torch.empty(n, P, dtype=torch.float64, device=F.device) if P else None
    ratio = torch.empty(n, P, dtype=torch.float64, device=F.device) if P else None
    _check(_lib.jtfs_knn_regress(_ptr(F), n, d, F.stride(0), _ptr(theta), P, K, _ptr(nbr), _ptr(hat), _ptr(ratio),
                                 _ptr(ws), ws.numel(), _stream_handle(stream)), "jtfs_knn_regress")
    return nbr, hat, ratio


def isomap(F, K: int = 40, n_components: int = 3, stream=None):
    """Isomap of feature rows F (float32 CUDA [n, d], row stride may exceed d).
    Returns (embedding float64 [n, n_components], eigenvalues float64 [n_components]).
    Synchronous; raises JTFSError if the K-NN graph is disconnected."""
    import torch
    assert F.dtype == torch.float32 and F.is_cuda and F.dim() == 2 and F.stride(1) == 1
    n, d = F.shape
    sz = C.c_size_t()
    _check(_lib.jtfs_isomap_workspace_size(n, K, C.byref(sz)), "jtfs_isomap_workspace_size")
    ws = torch.empty(max(int(sz.value), 1), dtype=torch.uint8, device=F.device)
    emb = torch.empty(n, n_components, dtype=torch.float64, device=F.device)
    ev = torch.empty(n_components, dtype=torch.float64, device=F.device)
    _check(_lib.jtfs_isomap(_ptr(F), n, d, F.stride(0), K, n_components, _ptr(emb), _ptr(ev), _ptr(ws), ws.numel(),
                            _stream_handle(stream)), "jtfs_isomap")
    return emb, ev


class UnitSet:
    """jtfs_unitset_create / jtfs_unitset_destroy."""

    def __init__(self, plan: "Plan", unit_ids):
        self.plan = plan            # keeps the plan alive while the set exists
        self.ids = [int(i) for i in unit_ids]
        arr = (C.c_int32 * max(len(self.ids), 1))(*self.ids)
        h = _P()
        _check(_lib.jtfs_unitset_create(plan.handle, arr, len(self.ids), C.byref(h)), "jtfs_unitset_create")
        self._h = h

    @property
    def handle(self):
        return self._h

    def __del__(self):
        try:
            if getattr(self, "_h", None):
                _lib.jtfs_unitset_destroy(self._h)
                self._h = None
        except Exception:
            pass


def measure_fp32_peak(device: int = 0):
    """(FFMA, FFMA2) TFLOP/s measured on `device` (jtfs_measure_fp32_peak; synchronous)."""
    a, b = C.c_double(), C.c_double()
    _check(_lib.jtfs_measure_fp32_peak(device, C.byref(a), C.byref(b)), "jtfs_measure_fp32_peak")
    return a.value, b.value


def jtfs_plan(N, J, Q, J_fr, Q_fr, T, F, flags=0) -> Plan:
    """North-star form of jtfs.h's jtfs_plan (Q2 = 1, Eq. (3), reflect padding)."""
    return Plan(N=N, J=J, Q=Q, J_fr=J_fr, T=T, F=F, Q_fr=Q_fr, flags=flags)


def jtfs_forward(plan: Plan, x_batch, out=None, stream=None):
    """jtfs_forward(plan, x_batch, out) of jtfs.h."""
    return plan.forward(x_batch, out=out, stream=stream)
