"""CPU: host-side logic -- workload configs, algorithmic counts, argument
validation of the Python mirror, sharding arithmetic."""
import numpy as np
import pytest

from paper_1404_0424_b200 import CONFIGS, api, get_config
from paper_1404_0424_b200.parallel import shard_range


def test_configs_follow_reference_snr_conventions():
    c1 = get_config("cfg1")
    assert c1.n0 == pytest.approx(0.8) and c1.rho_u == pytest.approx(1.25)  # channel.cpp:44-47
    c3 = get_config("cfg3")
    assert c3.n0 == pytest.approx(0.1) and c3.rho_d == pytest.approx(0.625)  # channel.cpp:49-51
    c5 = get_config("cfg5")
    assert c5.rho_d == pytest.approx(c5.rho_u)  # A_dl == A_ul: the Gram is shared
    assert c5.rsqrt().shape == (256, 256)
    R = 0.5 ** np.abs(np.subtract.outer(np.arange(256), np.arange(256)))
    np.testing.assert_allclose(c5.rsqrt() @ c5.rsqrt(), R, atol=1e-10)


def test_algorithmic_counts_match_survey_table():
    # flop / byte per vector
    want = {"cfg1": (56192, 9472), "cfg2": (112795, 4645), "cfg3": (163328, 17540),
            "cfg5": (850112, 9732), "cfg4a_K2": (596800, 18176), "cfg4b_K8": (11264128, 69120)}
    for name, (f, b) in want.items():
        c = CONFIGS[name]
        assert round(c.flops_per_vector()) == f, name
        assert round(c.bytes_per_vector()) == b, name


def test_argument_validation_mirrors_reference():
    H = np.zeros((2, 8, 4), np.complex64)
    assert api.detect_dims(H, np.zeros((2, 8, 3), np.complex64)) == (2, 8, 4, 3)
    with pytest.raises(ValueError):
        api.detect_dims(H, np.zeros((2, 7, 3), np.complex64))
    with pytest.raises(ValueError):
        api.detect_dims(H[0], np.zeros((8, 3), np.complex64))
    Hd = np.zeros((2, 4, 16), np.complex64)
    assert api.precode_dims(Hd, np.zeros((2, 5, 4), np.complex64)) == (2, 16, 4, 5)
    assert api.precode_dims(H, np.zeros((2, 1, 4), np.complex64), uplink_layout=True) == (2, 8, 4, 1)
    with pytest.raises(ValueError):
        api.precode_dims(Hd, np.zeros((2, 5, 3), np.complex64))
    with pytest.raises(ValueError):
        api._check_inputs(False, np.zeros((2, 3), np.complex128))
    with pytest.raises(ValueError):
        api.detect_cg_single(np.zeros((8, 4)), np.zeros(7), 1.0, 1.0, 1.0, 4, 2)


@pytest.mark.parametrize("n,w", [(1200, 1), (1200, 2), (1200, 8), (65536, 8), (7, 4), (3, 8)])
def test_shard_range_partitions_contiguously(n, w):
    spans = [shard_range(n, r, w) for r in range(w)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_seed_scheme_is_shard_invariant(oracle_port):
    """Per-subcarrier streams (root.fork(2).fork(sc)) make any shard's inputs
    identical to the same rows of the unsharded draw."""
    full = [oracle_port.rayleigh(3, [2, sc], 16, 4) for sc in range(12)]
    for w in (2, 3, 4):
        for r in range(w):
            a, b = shard_range(12, r, w)
            part = [oracle_port.rayleigh(3, [2, sc], 16, 4) for sc in range(a, b)]
            assert all(np.array_equal(x, y) for x, y in zip(part, full[a:b]))


def test_output_buffers_are_validated():
    """Caller-supplied out= buffers: wrong shape, dtype, layout or memory
    space raise ValueError before any pointer reaches the C ABI."""
    like = np.zeros((2, 8, 4), np.complex64)
    shapes = {"mu": ((2, 3, 4), "f32"), "xhat": ((2, 3, 4), "c64")}
    api._check_outputs({"mu": np.zeros((2, 3, 4), np.float32)}, shapes, False, like)
    with pytest.raises(ValueError):  # undersized
        api._check_outputs({"mu": np.zeros((2, 3, 3), np.float32)}, shapes, False, like)
    with pytest.raises(ValueError):  # dtype
        api._check_outputs({"mu": np.zeros((2, 3, 4), np.float64)}, shapes, False, like)
    with pytest.raises(ValueError):  # not contiguous
        api._check_outputs({"xhat": np.zeros((2, 4, 3), np.complex64).transpose(0, 2, 1)},
                           shapes, False, like)
    with pytest.raises(ValueError):  # a host array in a device call
        import torch

        api._check_outputs({"mu": np.zeros((2, 3, 4), np.float32)}, shapes, True,
                           torch.zeros(1))
    with pytest.raises(ValueError):  # unknown name
        api._check_outputs({"nu": np.zeros((2, 3, 4), np.float32)}, shapes, False, like)


def test_precoder_rotation_table_matches_its_bank_model():
    """The start rotations compiled into precode_small_kernel (U = 16,
    64-antenna chunks) are valid for their lanes' pair ranges and keep the
    Gram loads' modelled wavefront count within 10 % of conflict-free, well
    below the unsearched start (tools/ps_rotation.py holds the model)."""
    import importlib.util
    import os
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("ps_rotation", os.path.join(root, "tools", "ps_rotation.py"))
    psr = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(psr)
    src = open(os.path.join(root, "paper_1404_0424_b200", "csrc", "cgm_precode_small.cuh")).read()
    m = re.search(r"kRot\[32\] = \{([^}]*)\}", src)
    assert m, "rotation table not found"
    rot = [int(x) for x in m.group(1).replace("\n", " ").split(",")]
    assert len(rot) == 32
    for lane, L in enumerate(psr.lanes):
        if L is not None:
            assert 0 <= rot[lane] < L[3], (lane, rot[lane], L[3])
    ideal = 88  # 11 steps x 4 quarter-warp phases x (x, y loads), one wavefront each
    assert psr.cost(rot) <= 1.1 * ideal
    assert psr.cost(psr.baseline()) > 1.5 * psr.cost(rot)


def test_uplink_small_gram_loads_are_conflict_free_in_the_bank_model():
    """uplink_small_kernel's full-U Gram loop (cfg1, U = 8; also U = 16):
    strided antenna parts with the pair order rot2 the kernel compiles in give
    one wavefront per quarter-warp LDS.128, where the unrotated order needs up
    to two (tools/us_rotation.py holds the model; rot2 read from the source)."""
    import importlib.util
    import os
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("us_rotation", os.path.join(root, "tools", "us_rotation.py"))
    usr = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(usr)
    src = open(os.path.join(root, "paper_1404_0424_b200", "csrc", "cgm_uplink_small.cuh")).read()
    # the model's rot2_of must be the kernel's expression
    assert re.search(r"rot2 = p\.U != UP \? 0 : UP == 8 \? \(item_part >> 1\) & 1 : item_part & 1;", src)
    for UP in (8, 16):
        worst, mean = usr.wavefronts(UP)
        assert worst == 1 and mean == 1.0, (UP, worst, mean)
        worst0, mean0 = usr.wavefronts(UP, rotate=False)
        assert worst0 == 2 and mean0 > 1.2, (UP, worst0, mean0)
