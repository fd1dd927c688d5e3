"""GPU: whole-configuration parity against the unmodified reference --
every instance of cfg1 / cfg2 / cfg3 and 4096 subcarriers (all vectors) of
cfg4a / cfg4b (K = 2, 4, 8) and cfg5 (tests/parity_full.py; the committed
report is profiles/r02_parity.json), plus BASELINE configs[3]'s CG-K vs
exact-MMSE error comparison computed on the GPU and on the reference."""
import pytest

import parity_full

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def report(oracle_ref):
    return parity_full.run()


def test_every_checked_instance_within_contract(report):
    assert parity_full.failures(report) == []


def test_exact_mmse_error_tables_agree(report):
    """The CG-K error against exact MMSE is the same quantity whether the GPU
    (CG vs Cholesky kernels) or the reference (detect_cg vs detect_explicit)
    computes it."""
    for name, sec in report["configs"].items():
        if not name.startswith("cfg4"):
            continue
        m = sec["vs_exact_mmse"]
        for k in ("xhat_rel_err_median", "rho_rel_err_median"):
            assert m["agreement"][k] < 0.05, (name, k, m["gpu"][k], m["reference"][k])
        g, r = m["gpu"]["hard_bit_disagreement"], m["reference"]["hard_bit_disagreement"]
        assert abs(g - r) <= 0.1 * r + 1e-4, (name, g, r)
        for k, v in m["exact_mmse_gpu_vs_reference"].items():
            assert v["outside_tol"] == 0, (name, "exact MMSE", k, v)
