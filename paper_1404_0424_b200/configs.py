"""The BASELINE.json workloads as data.

SNR conventions follow the reference: uplink N0 = U Es / SNR
(channel.cpp:44-47) and rho_u = Es / N0 (sim.cpp:376-377); downlink
N0 = 1 / SNR (channel.cpp:49-51) with the BASELINE regulariser alpha = U N0 / Es,
passed to precode_cg as rho_d = 1 / alpha (the reference harness uses
alpha = N0, sim.cpp:397-398 -- only the argument differs).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    kind: str              # "uplink" | "downlink" | "both"
    B: int
    U: int
    S: int                 # vectors per subcarrier sharing H
    n_sc: int
    K: int
    tracker: str = "exact"
    qam_bits: int = 6
    snr_db: float = 15.0
    seed: int = 1
    corr: float = 0.0      # BS-side exponential correlation R_ij = corr^|i-j|
    es: float = 1.0

    @property
    def n0(self) -> float:
        snr = 10.0 ** (self.snr_db / 10.0)
        return self.U * self.es / snr if self.kind != "downlink" else 1.0 / snr

    @property
    def rho_u(self) -> float:
        return self.es / self.n0

    @property
    def rho_d(self) -> float:
        snr = 10.0 ** (self.snr_db / 10.0)
        alpha = self.U * (1.0 / snr) / self.es
        return 1.0 / alpha

    @property
    def vectors(self) -> int:
        return self.n_sc * self.S

    # ---- algorithmic counts of SURVEY.md section 8(d) (complex MAC = 8 flops,
    # Hermitian products on one triangle, each input read once / output
    # written once; intermediates not credited)
    def flops_per_vector(self) -> float:
        B, U, K, S = self.B, self.U, self.K, self.S
        M = 1 << self.qam_bits
        f = 0.0
        if self.kind in ("uplink", "both"):
            f += 4 * B * U * (U + 1) / S                    # Gram, shared by S vectors
            f += 8 * B * U                                  # matched filter
            f += K * (8 * U * U + 20 * U) + 4 * U           # CG
            if self.tracker == "exact":
                f += (K - 1) * 4 * U * (U + 1) * (U + 2) + 4 * U * U * (U + 1) + 8 * U * U
            else:
                f += (K - 1) * 6 * U + 2 * U
            f += U * (4 + self.qam_bits * (3 * np.sqrt(M) + 3))  # LLR
        if self.kind == "downlink":
            f += 4 * B * U * (U + 1) / S
        if self.kind in ("downlink", "both"):
            f += K * (8 * U * U + 20 * U) + 4 * U + 8 * B * U + 4 * B
        return f

    def bytes_per_vector(self) -> float:
        B, U, S = self.B, self.U, self.S
        b = 8 * B * U / S                                   # channel, shared by S vectors
        if self.kind in ("uplink", "both"):
            b += 8 * B + 8 * U + 4 * U + 4 * U + 4 * U * self.qam_bits
        if self.kind in ("downlink", "both"):
            b += 8 * U + 8 * B + 4
        return b

    # ---- the same counts split by kernel (bench.py's per-kernel rooflines)
    def channel_flops_per_vector(self) -> float:
        """Gram (+ matched filter) of the channel kernel."""
        B, U, S = self.B, self.U, self.S
        f = 4 * B * U * (U + 1) / S
        if self.kind in ("uplink", "both"):
            f += 8 * B * U
        return f

    def channel_bytes_per_vector(self) -> float:
        """H (shared by S vectors) + y read by the channel kernel."""
        b = 8 * self.B * self.U / self.S
        if self.kind in ("uplink", "both"):
            b += 8 * self.B
        return b

    def tracker_basis_flops_per_vector(self) -> float:
        """The exact tracker's U^3 recursion, (K-1) 4U(U+1)(U+2) per VECTOR in
        the reference (detect.cpp:336-368) -- part of flops_per_vector."""
        if self.kind not in ("uplink", "both") or self.tracker != "exact":
            return 0.0
        U, K = self.U, self.K
        return (K - 1) * 4 * U * (U + 1) * (U + 2)

    def tracker_extract_flops_per_vector(self) -> float:
        """The exact tracker's extraction (detect.cpp:370-395), per vector."""
        if self.kind not in ("uplink", "both") or self.tracker != "exact":
            return 0.0
        U = self.U
        return 4 * U * U * (U + 1) + 8 * U * U

    def basis_flops_per_vector(self) -> float:
        """What the moments kernel (cgm_moments.cuh) does: the same (K-1)
        Hermitian products once per SUBCARRIER, shared by its S vectors."""
        return self.tracker_basis_flops_per_vector() / self.S

    def solve_flops_per_vector(self) -> float:
        """CG, tracker extraction, LLRs (+ precoder): the rest of the path."""
        return (self.flops_per_vector() - self.channel_flops_per_vector()
                - self.tracker_basis_flops_per_vector())

    def moments_extract_flops_per_vector(self) -> float:
        """The row-moment extraction this repo runs per vector (cgm_moments.cuh):
        two Chebyshev coefficient products (~4 K^2) and, per user row, four
        dot products of length <= 2K + 1 (8 (2K + 1) flops)."""
        if self.kind not in ("uplink", "both") or self.tracker != "exact":
            return 0.0
        K, U = self.K, self.U
        return 4 * K * K + 8 * (2 * K + 1) * U

    def solve_kernel_flops_per_vector(self) -> float:
        """What the solve kernel computes: CG, LLRs (+ precoder) and the
        moment extraction in place of the reference's U^3 extraction."""
        return (self.solve_flops_per_vector() - self.tracker_extract_flops_per_vector()
                + self.moments_extract_flops_per_vector())

    def precoder_flops_per_vector(self) -> float:
        """q = H_d^H v (8 B U) and the gain ||q|| (4 B) of a transmit vector --
        the separate precoder kernel of detect + precode calls (cgm_block32.cuh)."""
        return 8 * self.B * self.U + 4 * self.B if self.kind == "both" else 0.0

    def precoder_bytes_per_vector(self) -> float:
        """H re-read (shared by S vectors), v_K in, q and s out, gain + status."""
        if self.kind != "both":
            return 0.0
        return 8 * self.B * self.U / self.S + 8 * self.U + 16 * self.B + 5

    def solve_bytes_per_vector(self, precoder_separate: bool = False) -> float:
        """Bytes of the solve kernel: the path's bytes minus the channel
        kernel's; with the precoder as its own kernel (detect + precode
        calls) only the uplink outputs and the transmit vector read."""
        if precoder_separate and self.kind == "both":
            U = self.U
            return 8 * U + 4 * U + 4 * U + 4 * U * self.qam_bits + 8 * U
        return self.bytes_per_vector() - self.channel_bytes_per_vector()

    def scaled(self, n_sc: int) -> "Config":
        return replace(self, n_sc=n_sc)

    def rsqrt(self) -> np.ndarray | None:
        """R^{1/2} of R_ij = corr^|i-j| (B x B), FP64 symmetric eigendecomposition."""
        if not self.corr:
            return None
        idx = np.arange(self.B)
        R = self.corr ** np.abs(idx[:, None] - idx[None, :])
        w, V = np.linalg.eigh(R)
        return (V * np.sqrt(np.clip(w, 0.0, None))) @ V.T


CONFIGS = {
    "cfg1": Config("cfg1", "uplink", B=128, U=8, S=1, n_sc=1024, K=3, tracker="exact",
                   qam_bits=4, snr_db=10.0, seed=1),
    "cfg2": Config("cfg2", "uplink", B=128, U=32, S=14, n_sc=1200, K=4, tracker="approx",
                   qam_bits=6, snr_db=15.0, seed=2),
    "cfg3": Config("cfg3", "downlink", B=128, U=16, S=1, n_sc=16384, K=3, qam_bits=4,
                   snr_db=10.0, seed=3),
    "cfg5": Config("cfg5", "both", B=256, U=32, S=16, n_sc=65536, K=4, tracker="exact",
                   qam_bits=6, snr_db=15.0, seed=5, corr=0.5),
}
for _K in (2, 4, 8):
    CONFIGS[f"cfg4a_K{_K}"] = Config(f"cfg4a_K{_K}", "uplink", B=64, U=32, S=1, n_sc=65536,
                                     K=_K, tracker="exact", qam_bits=6, snr_db=20.0, seed=4)
    CONFIGS[f"cfg4b_K{_K}"] = Config(f"cfg4b_K{_K}", "uplink", B=128, U=64, S=1, n_sc=65536,
                                     K=_K, tracker="exact", qam_bits=6, snr_db=20.0, seed=4)


def get_config(name: str) -> Config:
    return CONFIGS[name]
