"""NEXT-3 on the CUDA path: the paper's simulation suite (Fig. 4 data sets of section 4.2.1, P:331;
Appendix A overlap frames) against the oracle -- exact (equal K, labels up to a bijection,
centres within 1e-4, identical per-round traces), and the generator's truth recovered."""
import numpy as np
import pytest

from synth.frames import make_circles, make_overlap, make_polarized
from tests.parity_util import bijection
from tests.test_gpu_parity import check_exact

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_circles_fixed64_exact(seed):
    x, t = make_circles(seed)
    lg, cg, Kg, st, ro = check_exact(x, kind=0, n_seeds=64, rng_seed=seed, has_background=0)
    if ro.K == 10:
        assert bijection(lg[0], t)


@pytest.mark.parametrize("instances", [7, 3])
def test_polarized_osop_exact(instances):
    x, t = make_polarized(0, instances)
    lg, cg, Kg, st, ro = check_exact(x, n_seeds=64, rng_seed=2)
    assert Kg[0] == instances + 1 and bijection(lg[0], t)
    assert st["frames"][0]["round_r"][-1] == 0.5


@pytest.mark.parametrize("spacing", [300, 150])
def test_appendix_a_overlap_exact(spacing):
    """1000 x 1000 x 18 (32-lane operand rows), P = 0.95 (R16)."""
    x, t = make_overlap(spacing)
    lg, cg, Kg, st, ro = check_exact(x, P=0.95, rng_seed=0)
    assert Kg[0] == 9 and bijection(lg[0], t)
