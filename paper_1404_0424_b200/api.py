"""Host-side mirror of the reference's detector / precoder interface.

Same names, argument meaning and error behaviour as the reference's
``cgmimo::detect::detect_cg`` (detect.hpp:58-61) and
``cgmimo::precode::precode_cg`` (precode.hpp:31-33), batched:

* ``H`` uplink ``(n_sc, B, U)`` complex64, ``Y`` ``(n_sc, B, S)`` complex64
  (antenna-major: column s is the s-th received vector sharing channel
  ``sc``); downlink ``Hd`` ``(n_sc, U, B)``,
  ``T`` ``(n_sc, S, U)``.
* numpy arrays are HOST buffers (synchronous call, copies pipelined inside the
  C ABI); torch CUDA tensors are DEVICE buffers (asynchronous on the current
  torch stream).
* bad arguments raise ``ValueError`` (the reference's std::invalid_argument);
  a per-instance solver breakdown is reported in ``status`` (bit 0) like the
  batched C ABI, and ``detect_cg_single`` / ``precode_cg_single`` raise
  ``SolverBreakdown`` like the reference's per-call API.
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib

TRACKERS = {"exact": _lib.CGM_TRACKER_EXACT, "approx": _lib.CGM_TRACKER_APPROX}


class SolverBreakdown(RuntimeError):
    """Non-positive curvature p^H A p (reference solvers.cpp:55-57)."""


class CudaError(RuntimeError):
    pass


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _ptr(x):
    if x is None:
        return None
    if _is_torch(x):
        return C.c_void_p(x.data_ptr())
    return x.ctypes.data_as(C.c_void_p)


class Context:
    """One C-ABI context (device, stream, workspaces).  Not thread-safe: use one
    per host thread (``default_context()`` is thread-local)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        rc = self.lib.cgm_ctx_create(int(device), C.byref(h))
        if rc != _lib.CGM_OK:
            raise CudaError(f"cgm_ctx_create(device={device}) failed rc={rc}: no usable sm_100 GPU")
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self.lib.cgm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------- helpers
    def _check(self, rc: int):
        if rc == _lib.CGM_OK:
            return
        msg = self.lib.cgm_last_error(self.h).decode()
        if rc == _lib.CGM_EINVAL:
            raise ValueError(msg)
        raise CudaError(f"rc={rc}: {msg}")

    def set_stream(self, stream_handle: int):
        self._check(self.lib.cgm_ctx_set_stream(self.h, C.c_void_p(stream_handle)))

    def _bind_torch_stream(self):
        import torch

        self.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    POLICY_FLAGS = {"ffma_channel": 1, "split_small": 2, "lane_solve": 4, "block_uplink": 8,
                    "rows_cta": 16, "poison_ws": 32, "tile_moments": 64, "serial_chunks": 128,
                    "untiled_cg": 256, "pairs_cg": 512}

    def set_kernel_policy(self, policy: str):
        """Kernel-variant switches for A/B tests: "auto" (production defaults)
        or "+"-joined names of POLICY_FLAGS -- "ffma_channel" (FFMA Gram
        kernel instead of tcgen05 for U = 32), "split_small" (channel + solve
        pair instead of the fused U <= 16 kernels), "lane_solve" (lane-per-row
        solve kernel instead of the U = 32 row kernels), "block_uplink" (the
        shared-G block kernel for U = 32 uplink-only calls instead of the pairs
        kernel), "rows_cta" (the 8-warp row CTA instead of the block kernel
        for calls with transmit vectors), "poison_ws" (test only: NaN-fill the
        workspace before every chunk), "tile_moments" (the 4x4-tile CTA
        moments kernel instead of the warp-per-subcarrier one, U = 32),
        "serial_chunks" (every workspace chunk on the call's stream instead of
        alternating two streams), "untiled_cg" (the lane-per-row 8-warp block
        CG kernel instead of the register-tiled one for the exact tracker with
        transmit vectors, cfg5), "pairs_cg" (the warp-per-pair-of-systems
        kernel with the Gram row in registers instead of the register-tiled
        block CG for approximate-tracker uplink calls, cfg2)."""
        bits = 0
        if policy != "auto":
            for name in policy.split("+"):
                bits |= self.POLICY_FLAGS[name]
        self._check(self.lib.cgm_ctx_set_kernel_policy(self.h, bits))

    def set_profiling(self, on: bool):
        self._check(self.lib.cgm_ctx_set_profiling(self.h, 1 if on else 0))

    def kernel_times_ex(self):
        """(channel_ms, moments_ms, solve_ms, launches) summed since profiling
        was enabled; moments = the exact tracker's row-moment kernel."""
        a, b, c, n = C.c_double(), C.c_double(), C.c_double(), C.c_long()
        self._check(self.lib.cgm_ctx_kernel_times_ex(self.h, C.byref(a), C.byref(b), C.byref(c),
                                                     C.byref(n)))
        return a.value, b.value, c.value, n.value

    def kernel_times_kinds(self):
        """({"channel", "moments", "solve", "precoder"}: ms, launches) summed since
        profiling was enabled (the precoder kernel separate from the solve)."""
        ms = (C.c_double * 4)()
        n = C.c_long()
        self._check(self.lib.cgm_ctx_kernel_times_kinds(self.h, ms, C.byref(n)))
        return dict(zip(("channel", "moments", "solve", "precoder"), list(ms))), n.value

    def kernel_timeline(self, cap: int = 4096):
        """[(kind, start_ms, end_ms)] of the launches recorded since profiling
        was enabled (kind: "channel" / "solve" / "moments" / "precoder"),
        relative to the first one's start."""
        k = (C.c_int * cap)()
        a = (C.c_double * cap)()
        b = (C.c_double * cap)()
        n = C.c_long()
        self._check(self.lib.cgm_ctx_kernel_timeline(self.h, k, a, b, cap, C.byref(n)))
        names = {1: "channel", 2: "solve", 3: "moments", 4: "precoder"}
        return [(names.get(k[i], str(k[i])), a[i], b[i]) for i in range(min(n.value, cap))]

    def kernel_times(self):
        """(channel_ms, solve_ms, launches) summed since profiling was enabled."""
        a, b, n = C.c_double(), C.c_double(), C.c_long()
        self._check(self.lib.cgm_ctx_kernel_times(self.h, C.byref(a), C.byref(b), C.byref(n)))
        return a.value, b.value, n.value

    def synchronize(self):
        self._check(self.lib.cgm_synchronize(self.h))

    @property
    def kernel_launches(self) -> int:
        return int(self.lib.cgm_kernel_launches(self.h))

    # ------------------------------------------------- coded BLER harness
    def uplink_trials(self, B, U, n_sc, qam_bits, K, tracker, snr_db, trial_keys):
        """cgm_uplink_trials: block errors and breakdown flags of a batch of
        the reference's coded uplink trials (sim.cpp:147-203)."""
        import numpy as np

        keys = np.ascontiguousarray(trial_keys, dtype=np.uint64)
        n = len(keys)
        errs = np.zeros(n, np.uint32)
        brk = np.zeros(n, np.uint8)
        trk = {"exact": _lib.CGM_TRACKER_EXACT, "approx": _lib.CGM_TRACKER_APPROX}[tracker]
        self._check(self.lib.cgm_uplink_trials(self.h, B, U, n_sc, qam_bits, K, trk, float(snr_db), n,
                                               keys.ctypes.data_as(C.c_void_p),
                                               errs.ctypes.data_as(C.c_void_p),
                                               brk.ctypes.data_as(C.c_void_p)))
        return errs, brk

    def downlink_trials(self, B, U, n_sc, qam_bits, K, snr_db, trial_keys):
        """cgm_downlink_trials: block errors and breakdown flags of a batch of
        the reference's coded downlink trials (sim.cpp:205-275)."""
        import numpy as np

        keys = np.ascontiguousarray(trial_keys, dtype=np.uint64)
        n = len(keys)
        errs = np.zeros(n, np.uint32)
        brk = np.zeros(n, np.uint8)
        self._check(self.lib.cgm_downlink_trials(self.h, B, U, n_sc, qam_bits, K, float(snr_db), n,
                                                 keys.ctypes.data_as(C.c_void_p),
                                                 errs.ctypes.data_as(C.c_void_p),
                                                 brk.ctypes.data_as(C.c_void_p)))
        return errs, brk

    def viterbi_decode(self, llrs):
        """cgm_viterbi_decode: (n_cw, coded_len) float64 LLRs -> (n_cw, info_len) bits."""
        import numpy as np

        llrs = np.ascontiguousarray(np.atleast_2d(llrs), dtype=np.float64)
        n_cw, coded = llrs.shape
        out = np.zeros((n_cw, coded // 6 * 5 - 6), np.uint8)
        self._check(self.lib.cgm_viterbi_decode(self.h, llrs.ctypes.data_as(C.c_void_p), coded, n_cw,
                                                out.ctypes.data_as(C.c_void_p)))
        return out

    # ------------------------------------------------------------- detect
    def detect(self, method, H, Y, rho_u, n0, es, qam_bits, iters=1, tracker="approx", out=None,
               want=("xhat", "mu", "rho", "llr", "status")):
        """Batched detect_<method> (cgm_detect): method "cholesky" (alias
        "chol"), "cg", "cgls" or "neumann" (iters = series terms)."""
        if method not in _lib.METHODS:
            raise ValueError(f"unknown method {method!r}")
        return self.detect_cg(H, Y, rho_u, n0, es, qam_bits, iters, tracker, out, want,
                              method=method)

    def detect_cg(self, H, Y, rho_u, n0, es, qam_bits, iters, tracker="exact", out=None,
                  want=("xhat", "mu", "rho", "llr", "status"), method="cg"):
        """Batched detect_cg.  Returns dict with the requested outputs."""
        device = _is_torch(H)
        n_sc, B, U, S = detect_dims(H, Y)
        if tracker not in TRACKERS:
            raise ValueError(f"unknown tracker {tracker!r}")
        out = dict(out or {})
        shapes = {"xhat": ((n_sc, S, U), "c64"), "mu": ((n_sc, S, U), "f32"),
                  "rho": ((n_sc, S, U), "f32"), "llr": ((n_sc, S, U, qam_bits), "f32"),
                  "status": ((n_sc, S), "u8")}
        _check_outputs(out, shapes, device, H)
        for k in want:
            if k not in out:
                out[k] = _alloc(shapes[k], device, H)
        _check_inputs(device, H, Y)
        flags = 0
        if device:
            flags |= _lib.CGM_DEVICE_POINTERS
            self._bind_torch_stream()
        args = (B, U, n_sc, S, _ptr(H), _ptr(Y), float(rho_u), float(n0), float(es),
                int(qam_bits), int(iters), TRACKERS[tracker], _ptr(out.get("xhat")),
                _ptr(out.get("mu")), _ptr(out.get("rho")), _ptr(out.get("llr")),
                _ptr(out.get("status")), flags)
        if method == "cg":
            rc = self.lib.cgm_detect_cg(self.h, *args)
        else:
            rc = self.lib.cgm_detect(self.h, _lib.METHODS[method], *args)
        self._check(rc)
        return out

    # ------------------------------------------------------------ precode
    def precode(self, method, Hd, T, rho_d, iters=1, uplink_layout=False, out=None,
                want=("q", "s", "gain", "status")):
        """Batched precode_<method> (cgm_precode): "explicit" (Cholesky,
        alias "cholesky"), "cg", "cgls" or "neumann" (iters = series terms)."""
        if method not in _lib.METHODS:
            raise ValueError(f"unknown method {method!r}")
        return self.precode_cg(Hd, T, rho_d, iters, uplink_layout, out, want, method=method)

    def precode_cg(self, Hd, T, rho_d, iters, uplink_layout=False, out=None,
                   want=("q", "s", "gain", "status"), method="cg"):
        """Batched precode_cg.  Hd (n_sc, U, B); with uplink_layout=True the
        matrix is H_u (n_sc, B, U) and H_d = H_u^H (TDD reciprocity)."""
        device = _is_torch(Hd)
        n_sc, B, U, S = precode_dims(Hd, T, uplink_layout)
        out = dict(out or {})
        shapes = {"q": ((n_sc, S, B), "c64"), "s": ((n_sc, S, B), "c64"),
                  "gain": ((n_sc, S), "f32"), "status": ((n_sc, S), "u8")}
        _check_outputs(out, shapes, device, Hd)
        for k in want:
            if k not in out:
                out[k] = _alloc(shapes[k], device, Hd)
        _check_inputs(device, Hd, T)
        flags = _lib.CGM_HD_UPLINK_LAYOUT if uplink_layout else 0
        if device:
            flags |= _lib.CGM_DEVICE_POINTERS
            self._bind_torch_stream()
        args = (B, U, n_sc, S, _ptr(Hd), _ptr(T), float(rho_d), int(iters), _ptr(out.get("q")),
                _ptr(out.get("s")), _ptr(out.get("gain")), _ptr(out.get("status")), flags)
        if method == "cg":
            rc = self.lib.cgm_precode_cg(self.h, *args)
        else:
            rc = self.lib.cgm_precode(self.h, _lib.METHODS[method], *args)
        self._check(rc)
        return out

    def detect_precode_cg(self, H, Y, rho_u, n0, es, qam_bits, iters, tracker, T, rho_d, iters_t,
                          out=None, want=("xhat", "mu", "rho", "llr", "status", "q", "s", "gain",
                                          "pstatus")):
        """Uplink detection + downlink precoding on the same channels, one pass."""
        device = _is_torch(H)
        n_sc, B, U = H.shape
        if Y.ndim != 3 or Y.shape[:2] != (n_sc, B) or T.shape[0] != n_sc or T.shape[2] != U:
            raise ValueError("detect_precode_cg: dimension mismatch")
        S, St = Y.shape[2], T.shape[1]
        out = dict(out or {})
        shapes = {"xhat": ((n_sc, S, U), "c64"), "mu": ((n_sc, S, U), "f32"),
                  "rho": ((n_sc, S, U), "f32"), "llr": ((n_sc, S, U, qam_bits), "f32"),
                  "status": ((n_sc, S), "u8"), "q": ((n_sc, St, B), "c64"),
                  "s": ((n_sc, St, B), "c64"), "gain": ((n_sc, St), "f32"),
                  "pstatus": ((n_sc, St), "u8")}
        _check_outputs(out, shapes, device, H)
        for k in want:
            if k not in out:
                out[k] = _alloc(shapes[k], device, H)
        _check_inputs(device, H, Y, T)
        flags = 0
        if device:
            flags |= _lib.CGM_DEVICE_POINTERS
            self._bind_torch_stream()
        g = out.get
        rc = self.lib.cgm_detect_precode_cg(
            self.h, B, U, n_sc, S, _ptr(H), _ptr(Y), float(rho_u), float(n0), float(es),
            int(qam_bits), int(iters), TRACKERS[tracker], _ptr(g("xhat")), _ptr(g("mu")),
            _ptr(g("rho")), _ptr(g("llr")), _ptr(g("status")), St, _ptr(T), float(rho_d),
            int(iters_t), _ptr(g("q")), _ptr(g("s")), _ptr(g("gain")), _ptr(g("pstatus")), flags)
        self._check(rc)
        return out

    # ---------------------------------------------------------- generators
    def generate_uplink(self, B, U, n_sc, S, seed, qam_bits, n0, sc0=0, labels=False,
                        rsqrt=None):
        """Seeded device inputs (torch CUDA tensors): H (n_sc,B,U), Y (n_sc,B,S)."""
        import torch

        dev = torch.device("cuda", self.device)
        H = torch.empty((n_sc, B, U), dtype=torch.complex64, device=dev)
        Y = torch.empty((n_sc, B, S), dtype=torch.complex64, device=dev)
        L = torch.empty((n_sc, S, U), dtype=torch.uint8, device=dev) if labels else None
        self._bind_torch_stream()
        if rsqrt is None:
            rc = self.lib.cgm_generate_uplink(self.h, B, U, sc0, n_sc, S, seed, qam_bits,
                                              float(n0), _ptr(H), _ptr(Y), _ptr(L))
        else:
            R = rsqrt.to(device=dev, dtype=torch.float32).contiguous()
            rc = self.lib.cgm_generate_uplink_correlated(self.h, B, U, sc0, n_sc, S, seed,
                                                         qam_bits, float(n0), _ptr(R), _ptr(H),
                                                         _ptr(Y), _ptr(L))
        self._check(rc)
        return (H, Y, L) if labels else (H, Y)

    def generate_downlink(self, B, U, n_sc, S, seed, qam_bits, sc0=0, labels=False):
        import torch

        dev = torch.device("cuda", self.device)
        Hd = torch.empty((n_sc, U, B), dtype=torch.complex64, device=dev)
        T = torch.empty((n_sc, S, U), dtype=torch.complex64, device=dev)
        L = torch.empty((n_sc, S, U), dtype=torch.uint8, device=dev) if labels else None
        self._bind_torch_stream()
        self._check(self.lib.cgm_generate_downlink(self.h, B, U, sc0, n_sc, S, seed, qam_bits,
                                                   _ptr(Hd), _ptr(T), _ptr(L)))
        return (Hd, T, L) if labels else (Hd, T)

    def generate_symbols(self, U, n_sc, S, seed, qam_bits, sc0=0):
        import torch

        dev = torch.device("cuda", self.device)
        T = torch.empty((n_sc, S, U), dtype=torch.complex64, device=dev)
        self._bind_torch_stream()
        self._check(self.lib.cgm_generate_symbols(self.h, U, sc0, n_sc, S, seed, qam_bits,
                                                  _ptr(T), None))
        return T


def detect_dims(H, Y):
    """(n_sc, B, U, S) of a batched detect call; raises ValueError like the
    reference's std::invalid_argument (detect.cpp:186)."""
    if len(H.shape) != 3 or len(Y.shape) != 3:
        raise ValueError("detect_cg: H must be (n_sc, B, U) and Y (n_sc, B, S)")
    n_sc, B, U = H.shape
    if Y.shape[0] != n_sc or Y.shape[1] != B:
        raise ValueError("detect_cg: dimension mismatch")
    return n_sc, B, U, Y.shape[2]


def precode_dims(Hd, T, uplink_layout=False):
    """(n_sc, B, U, S) of a batched precode call (precode.cpp:60)."""
    if len(Hd.shape) != 3 or len(T.shape) != 3:
        raise ValueError("precode_cg: Hd must be (n_sc, U, B) and T (n_sc, S, U)")
    if uplink_layout:
        n_sc, B, U = Hd.shape
    else:
        n_sc, U, B = Hd.shape
    if T.shape[0] != n_sc or T.shape[2] != U:
        raise ValueError("precode_cg: dimension mismatch")
    return n_sc, B, U, T.shape[1]


def _alloc(spec, device, like):
    shape, kind = spec
    if device:
        import torch

        dt = {"c64": torch.complex64, "f32": torch.float32, "u8": torch.uint8}[kind]
        return torch.empty(shape, dtype=dt, device=like.device)
    dt = {"c64": np.complex64, "f32": np.float32, "u8": np.uint8}[kind]
    return np.empty(shape, dtype=dt)


_DT = {"c64": ("torch.complex64", np.complex64), "f32": ("torch.float32", np.float32),
       "u8": ("torch.uint8", np.uint8)}


def _check_outputs(out, shapes, device, like):
    """Every caller-supplied output buffer must have its array's shape and
    dtype, be C-contiguous, and live where the inputs live (a CUDA tensor on
    the inputs' device, or a host numpy array): the kernels write through the
    raw pointer (a host pointer in a device call poisons the
    context, an undersized buffer is written out of bounds)."""
    for k, a in out.items():
        if a is None:
            continue
        if k not in shapes:
            raise ValueError(f"unknown output {k!r}")
        shape, kind = shapes[k]
        if device:
            ok = (_is_torch(a) and a.is_cuda and a.device == like.device and a.is_contiguous()
                  and str(a.dtype) == _DT[kind][0])
        else:
            ok = (isinstance(a, np.ndarray) and a.dtype == _DT[kind][1] and a.flags.c_contiguous
                  and a.flags.writeable)
        if not ok:
            raise ValueError(f"output {k!r} must be a C-contiguous {kind} "
                             f"{'CUDA tensor on ' + str(like.device) if device else 'numpy array'}")
        if tuple(a.shape) != tuple(shape):
            raise ValueError(f"output {k!r} has shape {tuple(a.shape)}, expected {tuple(shape)}")


def _check_inputs(device, *arrs):
    for a in arrs:
        if device:
            if not (_is_torch(a) and a.is_cuda and a.is_contiguous()):
                raise ValueError("device inputs must be contiguous CUDA tensors")
            if str(a.dtype) != "torch.complex64":
                raise ValueError("inputs must be complex64")
        else:
            if not (isinstance(a, np.ndarray) and a.dtype == np.complex64 and a.flags.c_contiguous):
                raise ValueError("host inputs must be C-contiguous complex64 numpy arrays")


_tls = threading.local()


def default_context(device: int = 0) -> Context:
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ------------------------------------------------------- reference-shaped API
def detect_cg(H, Y, rho_u, n0, es, qam_bits, iters, tracker="exact", ctx=None, **kw):
    """Batched ``detect::detect_cg`` (reference detect.cpp:182-237)."""
    return (ctx or default_context(_device_of(H))).detect_cg(H, Y, rho_u, n0, es, qam_bits, iters,
                                                           tracker, **kw)


def precode_cg(Hd, T, rho_d, iters, ctx=None, **kw):
    """Batched ``precode::precode_cg`` (reference precode.cpp:56-71)."""
    return (ctx or default_context(_device_of(Hd))).precode_cg(Hd, T, rho_d, iters, **kw)


def detect_cg_single(h, y, rho_u, n0, es, qam_bits, iters, tracker="exact"):
    """Per-call form with the reference's exact semantics: h (B,U), y (B,)
    complex (any precision; converted to complex64); raises ValueError /
    SolverBreakdown.  Returns dict xhat (U,), mu, rho, llr (U, bits)."""
    h = np.asarray(h)
    y = np.asarray(y)
    if h.ndim != 2 or y.ndim != 1 or h.shape[0] != y.shape[0]:
        raise ValueError("detect_cg: dimension mismatch")
    H = np.ascontiguousarray(h, dtype=np.complex64)[None]
    Yb = np.ascontiguousarray(y, dtype=np.complex64)[None, :, None]
    o = detect_cg(H, Yb, rho_u, n0, es, qam_bits, iters, tracker)
    if o["status"][0, 0] & 1:
        raise SolverBreakdown("cg_solve: non-positive curvature p^H A p")
    return {k: v[0, 0] for k, v in o.items() if k != "status"}


def precode_cg_single(hd, t, rho_d, iters):
    """Per-call ``precode_cg``: hd (U,B), t (U,).  Returns dict precoded,
    transmit, gain, zero_input."""
    hd = np.asarray(hd)
    t = np.asarray(t)
    if hd.ndim != 2 or t.ndim != 1 or hd.shape[0] != t.shape[0]:
        raise ValueError("precode_cg: dimension mismatch")
    o = precode_cg(np.ascontiguousarray(hd, dtype=np.complex64)[None],
                   np.ascontiguousarray(t, dtype=np.complex64)[None, None], rho_d, iters)
    st = int(o["status"][0, 0])
    if st & 1:
        raise SolverBreakdown("cg_solve: non-positive curvature p^H A p")
    return dict(precoded=o["q"][0, 0], transmit=o["s"][0, 0], gain=float(o["gain"][0, 0]),
                zero_input=bool(st & 2))


def _device_of(x) -> int:
    if _is_torch(x) and x.is_cuda:
        return x.device.index or 0
    return 0
