"""oracle -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

Two FP64 CPU implementations of the reference hot path behind one numpy API:

* ``kind="ref"``  -- the UNMODIFIED reference library (``/root/reference/proj/src``)
  compiled by ``oracle/Makefile`` into ``oracle/_ref/libcgmimo_ref.so`` and driven
  through ``oracle/ref_shim.cpp`` (calls ``detect::detect_cg`` detect.cpp:182,
  ``precode::precode_cg`` precode.cpp:56, ... per instance).
* ``kind="port"`` -- ``oracle/cg_oracle.c``, the plain-C restatement (each function
  cites the reference file:line it follows), pinned against ``ref`` and the
  committed fixtures in ``tests/golden/``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(_HERE, "_ref", "libcgmimo_ref.so")
PORT_LIB = os.path.join(_HERE, "_build", "libcgoracle.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


def build(quiet: bool = True) -> None:
    """Compile the C restatement and, when the reference tree exists, oracle/_ref."""
    targets = ["port"]
    if os.path.isdir(REF_SRC):
        targets.append("ref")
        # the reference's sweep driver relinked against the product library
        # (needs paper_1404_0424_b200/libcgmimo_b200.so built first)
        if os.path.exists(os.path.join(_HERE, "..", "paper_1404_0424_b200", "libcgmimo_b200.so")):
            targets.append("relink")
    out = subprocess.run(["make", "-C", _HERE, "-j8", *targets], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def available(kind: str) -> bool:
    return os.path.exists(REF_LIB if kind == "ref" else PORT_LIB)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


class Oracle:
    """numpy front-end over one of the two oracle libraries."""

    def __init__(self, kind: str = "ref"):
        if kind not in ("ref", "port"):
            raise ValueError(kind)
        self.kind = kind
        path = REF_LIB if kind == "ref" else PORT_LIB
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        self.pfx = "ref_" if kind == "ref" else "orc_"
        self._threaded = kind == "ref"
        for nm in ("conv_encode", "viterbi_decode"):
            self._fn(nm).restype = C.c_long
        if kind == "ref":
            self.lib.ref_sweep.restype = C.c_long

    def _fn(self, name):
        return getattr(self.lib, self.pfx + name)

    # ------------------------------------------------------------ detection
    def detect(self, H, Y, rho_u, n0, es, qam_bits, K=1, tracker="approx", method="cg",
               threads=1):
        """H: (n_sc, B, U) complex; Y: (n_sc, B, S) complex (antenna-major, the
        product's batch layout; the S columns are the received vectors).
        Returns dict of arrays shaped (n_sc, S, U[, bits])."""
        H = _c128(H)
        n_sc, B, U = H.shape
        assert Y.shape[:2] == (n_sc, B), (Y.shape, H.shape)
        S = Y.shape[2]
        Y = _c128(np.transpose(Y, (0, 2, 1)))  # per-vector rows for the C entry points
        xhat = np.zeros((n_sc, S, U), np.complex128)
        mu = np.zeros((n_sc, S, U))
        rho = np.zeros((n_sc, S, U))
        llr = np.zeros((n_sc, S, U, qam_bits))
        status = np.zeros((n_sc, S), np.uint8)
        trk = 0 if tracker == "exact" else 1
        common_out = (_ptr(xhat), _ptr(mu), _ptr(rho), _ptr(llr), _ptr(status, _u8p))
        base = [C.c_int(B), C.c_int(U), C.c_long(n_sc), C.c_int(S), _ptr(H), _ptr(Y),
                C.c_double(rho_u), C.c_double(n0), C.c_double(es), C.c_int(qam_bits)]
        if method == "cg":
            f = self._fn("detect_cg")
            args = [*base, C.c_int(K), C.c_int(trk), *common_out]
        elif method == "explicit":
            f = self._fn("detect_explicit")
            args = [*base, *common_out]
        elif method in ("cholesky", "chol"):
            f = self._fn("detect_cholesky")
            args = [*base, *common_out]
        elif method in ("cgls", "neumann"):
            f = self._fn("detect_" + method)
            args = [*base, C.c_int(K), *common_out]
        else:
            raise ValueError(method)
        if self._threaded:
            args.append(C.c_int(threads))
        rc = f(*args)
        if rc != 0:
            raise ValueError(f"oracle detect rejected arguments (rc={rc})")
        return dict(xhat=xhat, mu=mu, rho=rho, llr=llr, status=status)

    # ------------------------------------------------------------ precoding
    def precode(self, Hd, T, rho_d, K=1, method="cg", threads=1):
        """Hd: (n_sc, U, B) complex; T: (n_sc, S, U) complex."""
        Hd = _c128(Hd)
        T = _c128(T)
        n_sc, U, B = Hd.shape
        S = T.shape[1]
        assert T.shape == (n_sc, S, U)
        q = np.zeros((n_sc, S, B), np.complex128)
        s = np.zeros((n_sc, S, B), np.complex128)
        gain = np.zeros((n_sc, S))
        status = np.zeros((n_sc, S), np.uint8)
        outs = (_ptr(q), _ptr(s), _ptr(gain), _ptr(status, _u8p))
        base = [C.c_int(B), C.c_int(U), C.c_long(n_sc), C.c_int(S), _ptr(Hd), _ptr(T),
                C.c_double(rho_d)]
        if method in ("cg", "cgls", "neumann"):
            args = [*base, C.c_int(K), *outs]
            f = self._fn("precode_" + method)
        elif method in ("explicit", "cholesky", "chol"):
            args = [*base, *outs]
            f = self._fn("precode_explicit")
        else:
            raise ValueError(method)
        if self._threaded:
            args.append(C.c_int(threads))
        f(*args)
        return dict(q=q, s=s, gain=gain, status=status)

    # ------------------------------------------------------------ helpers
    def compute_llrs(self, xhat: complex, mu: float, rho: float, qam_bits: int) -> np.ndarray:
        out = np.zeros(qam_bits)
        rc = self._fn("compute_llrs")(C.c_double(xhat.real), C.c_double(xhat.imag),
                                      C.c_double(mu), C.c_double(rho), C.c_int(qam_bits),
                                      _ptr(out))
        if rc:
            raise ValueError("bad qam_bits")
        return out

    def constellation(self, qam_bits: int):
        pts = np.zeros(1 << qam_bits, np.complex128)
        half = qam_bits // 2
        per = (1 << half) // 2
        a0 = np.zeros((half, per))
        a1 = np.zeros((half, per))
        self._fn("constellation")(C.c_int(qam_bits), _ptr(pts), _ptr(a0), _ptr(a1))
        return pts, a0, a1

    # ------------------------------------------------- coded BLER harness
    def _need_ref(self, what):
        if self.kind != "ref":
            raise NotImplementedError(f"{what}: reference library only (coding.cpp / sim.cpp)")

    def conv_encode(self, info) -> np.ndarray:
        """phy::conv_encode (coding.cpp): rate-5/6 punctured K=7 code."""
        info = np.ascontiguousarray(info, dtype=np.uint8)
        out = np.zeros(len(info) * 2 + 64, np.uint8)
        n = self._fn("conv_encode")(info.ctypes.data_as(C.c_void_p), C.c_long(len(info)),
                                     out.ctypes.data_as(C.c_void_p))
        if n < 0:
            raise ValueError("conv_encode: bad length")
        return out[:n]

    def viterbi_decode(self, llrs) -> np.ndarray:
        """phy::viterbi_decode_soft (coding.cpp): max-log soft Viterbi, FP64."""
        llrs = np.ascontiguousarray(llrs, dtype=np.float64)
        out = np.zeros(len(llrs), np.uint8)
        n = self._fn("viterbi_decode")(llrs.ctypes.data_as(C.c_void_p), C.c_long(len(llrs)),
                                        out.ctypes.data_as(C.c_void_p))
        if n < 0:
            raise ValueError("viterbi_decode: bad length")
        return out[:n]

    def make_interleaver(self, key: int, forks, n: int) -> np.ndarray:
        """phy::make_interleaver (coding.cpp) on Rng(key).fork(forks...)."""
        fk = np.ascontiguousarray(forks, dtype=np.uint64)
        perm = np.zeros(n, np.int64)
        self._fn("make_interleaver")(C.c_uint64(key), _ptr(fk, _u64p), C.c_int(len(fk)),
                                      C.c_long(n), perm.ctypes.data_as(C.c_void_p))
        return perm

    def uplink_sweep_point(self, B, U, qam_bits, K, tracker, snr_db, trials, n_sc, seed,
                           threads=0) -> dict:
        """sim::run_uplink_sweep (sim.cpp:365-384) at one SNR, CG detector:
        frames (user blocks), block_errors, breakdowns, trials_run."""
        self._need_ref("uplink_sweep_point")
        out = np.zeros(4, np.int64)
        rc = self.lib.ref_uplink_sweep_point(
            C.c_int(B), C.c_int(U), C.c_int(qam_bits), C.c_int(K),
            C.c_int(0 if tracker == "exact" else 1), C.c_double(snr_db), C.c_long(trials),
            C.c_long(n_sc), C.c_uint64(seed), C.c_int(threads), out.ctypes.data_as(C.c_void_p))
        if rc != 0:
            raise RuntimeError("run_uplink_sweep raised")
        return dict(zip(("frames", "block_errors", "breakdowns", "trials_run"), map(int, out)))

    def downlink_sweep_point(self, B, U, qam_bits, K, snr_db, trials, n_sc, seed,
                             threads=0) -> dict:
        """sim::run_downlink_sweep (sim.cpp:386-405) at one SNR, CG precoder."""
        self._need_ref("downlink_sweep_point")
        out = np.zeros(4, np.int64)
        rc = self.lib.ref_downlink_sweep_point(
            C.c_int(B), C.c_int(U), C.c_int(qam_bits), C.c_int(K), C.c_double(snr_db),
            C.c_long(trials), C.c_long(n_sc), C.c_uint64(seed), C.c_int(threads),
            out.ctypes.data_as(C.c_void_p))
        if rc != 0:
            raise RuntimeError("run_downlink_sweep raised")
        return dict(zip(("frames", "block_errors", "breakdowns", "trials_run"), map(int, out)))

    def sweep(self, direction, method, B, U, qam_bits, iters, tracker, snr_start, snr_stop,
              snr_step, trials, n_sc, seed, max_block_errors=0, max_breakdown_fraction=1.0,
              threads=0) -> list:
        """sim::run_uplink_sweep / run_downlink_sweep (sim.cpp:365-405) with
        any sim::Method: one dict per SNR point (SnrPointResult fields)."""
        self._need_ref("sweep")
        out = np.zeros((256, 9))
        m = {"chol": 0, "cholesky": 0, "cg": 1, "cgls": 2, "neumann": 3}[method]
        n = self.lib.ref_sweep(
            C.c_int({"uplink": 1, "downlink": 2}[direction]), C.c_int(m), C.c_int(B), C.c_int(U),
            C.c_int(qam_bits), C.c_int(iters), C.c_int(0 if tracker == "exact" else 1),
            C.c_double(snr_start), C.c_double(snr_stop), C.c_double(snr_step), C.c_long(trials),
            C.c_long(n_sc), C.c_uint64(seed), C.c_long(max_block_errors),
            C.c_double(max_breakdown_fraction), C.c_int(threads), out.ctypes.data_as(C.c_void_p),
            C.c_long(256))
        if n < 0:
            raise RuntimeError({-1: "ConfigError", -2: "BreakdownBudgetExceeded"}.get(n, "error"))
        keys = ("snr_db", "frames", "block_errors", "bler", "bler_lo", "bler_hi",
                "real_mults_mean", "breakdowns", "trials_run")
        return [dict(zip(keys, row)) for row in out[:n]]

    def tradeoff_row(self, method, B, U, iters, snr, frames, errors, target):
        """sim::tradeoff_table for one sweep -> (real_mults, snr_at_target or None)."""
        self._need_ref("tradeoff_row")
        m = {"chol": 0, "cholesky": 0, "cg": 1, "cgls": 2, "neumann": 3}[method]
        snr = np.ascontiguousarray(snr, dtype=np.float64)
        fr = np.ascontiguousarray(frames, dtype=np.uint64)
        er = np.ascontiguousarray(errors, dtype=np.uint64)
        rm = C.c_uint64(0)
        st = C.c_double(0.0)
        ok = self.lib.ref_tradeoff_row(C.c_int(m), C.c_int(B), C.c_int(U), C.c_int(iters),
                                       snr.ctypes.data_as(C.c_void_p), fr.ctypes.data_as(C.c_void_p),
                                       er.ctypes.data_as(C.c_void_p), C.c_long(len(snr)),
                                       C.c_double(target), C.byref(rm), C.byref(st))
        return int(rm.value), (st.value if ok else None)

    def wilson(self, errors, total):
        self._need_ref("wilson")
        lo, hi = C.c_double(0), C.c_double(0)
        self.lib.ref_wilson(C.c_uint64(errors), C.c_uint64(total), C.byref(lo), C.byref(hi))
        return lo.value, hi.value

    def rng_u64(self, key: int, forks, n: int) -> np.ndarray:
        fk = np.ascontiguousarray(forks, dtype=np.uint64)
        out = np.zeros(n, np.uint64)
        self._fn("rng_u64")(C.c_uint64(key), _ptr(fk, _u64p), C.c_int(len(fk)), C.c_long(n),
                            _ptr(out, _u64p))
        return out

    def rng_cgaussian(self, key: int, forks, variance: float, n: int) -> np.ndarray:
        fk = np.ascontiguousarray(forks, dtype=np.uint64)
        out = np.zeros(n, np.complex128)
        self._fn("rng_cgaussian")(C.c_uint64(key), _ptr(fk, _u64p), C.c_int(len(fk)),
                                  C.c_double(variance), C.c_long(n), _ptr(out))
        return out

    def rayleigh(self, key: int, forks, B: int, U: int) -> np.ndarray:
        fk = np.ascontiguousarray(forks, dtype=np.uint64)
        out = np.zeros((B, U), np.complex128)
        self._fn("rayleigh")(C.c_uint64(key), _ptr(fk, _u64p), C.c_int(len(fk)), C.c_int(B),
                             C.c_int(U), _ptr(out))
        return out

    def gen_uplink(self, seed: int, B: int, U: int, sc0: int, n_sc: int, S: int,
                   qam_bits: int, n0: float, rsqrt=None, with_t: bool = False,
                   threads: int = 1):
        """The device generator's inputs (csrc/cgm_generate.cu) drawn on the host
        with the reference Rng: H (n_sc,B,U), Y (n_sc,B,S) [, T (n_sc,S,U)] complex64."""
        self._need_ref("gen_uplink")
        H = np.zeros((n_sc, B, U), np.complex64)
        Y = np.zeros((n_sc, B, S), np.complex64)
        T = np.zeros((n_sc, S, U), np.complex64) if with_t else None
        _fp = C.POINTER(C.c_float)
        R = None if rsqrt is None else np.ascontiguousarray(rsqrt, dtype=np.float32)
        rc = self.lib.ref_gen_uplink(C.c_uint64(seed), C.c_int(B), C.c_int(U), C.c_long(sc0),
                                     C.c_long(n_sc), C.c_int(S), C.c_int(qam_bits),
                                     C.c_double(n0), None if R is None else _ptr(R, _fp),
                                     _ptr(H, _fp), _ptr(Y, _fp),
                                     None if T is None else _ptr(T, _fp), C.c_int(threads))
        if rc != 0:
            raise ValueError("ref_gen_uplink: bad arguments")
        return (H, Y, T) if with_t else (H, Y)

    # reference-only probes ------------------------------------------------
    def count_detect_stages(self, method: int, B: int, U: int, K: int) -> np.ndarray:
        out = np.zeros(16, np.uint64)
        n = self.lib.ref_count_detect_stages(C.c_int(method), C.c_int(B), C.c_int(U),
                                             C.c_int(K), _ptr(out, _u64p))
        return out[:n]

    def tally_detect_cg(self, B: int, U: int, K: int, tracker: str, seed: int) -> np.ndarray:
        out = np.zeros(16, np.uint64)
        n = self.lib.ref_tally_detect_cg(C.c_int(B), C.c_int(U), C.c_int(K),
                                         C.c_int(0 if tracker == "exact" else 1),
                                         C.c_uint64(seed), _ptr(out, _u64p))
        return out[:n]

    def exact_filters(self, H, y, rho_u: float, K: int):
        H = _c128(H)
        y = _c128(y)
        B, U = H.shape
        filt = np.zeros((K, U, U), np.complex128)
        its = np.zeros((K, U), np.complex128)
        rc = self.lib.ref_exact_filters(C.c_int(B), C.c_int(U), _ptr(H), _ptr(y),
                                        C.c_double(rho_u), C.c_int(K), _ptr(filt), _ptr(its))
        if rc:
            raise RuntimeError(f"exact_filters rc={rc}")
        return filt, its
