"""The direct energy-resolving forward with register accumulators (option er_fwd_reg=1, the
default; csrc/operators.cu k_forward_reg): the same per-(pixel, energy) arithmetic in the
same order as the shared-memory-accumulator kernel (er_fwd_reg=0), so the bits agree; and
the oracle bar on energy counts that select each register-array size."""
import numpy as np
import pytest

import oracle
from workloads import make_config

torch = pytest.importorskip("torch")
P = pytest.importorskip("paper_1603_06400_b200")

from test_gpu_parity import assert_parity, gpu_forward, rnd  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ne", [8, 17, 40, 64, 100, 128])
def test_er_forward_registers_bitwise_and_oracle(ne):
    d = make_config(0, energy_resolving=1).desc()
    d.update(ne=ne, energy_kev=np.linspace(21.0, 149.0, ne), phi=np.linspace(1.0, 0.3, ne),
             ny=6, nz=5, nq=21, det_nx=7, det_ny=19)
    G = P.Geometry(d)
    f = rnd(G.f_shape, 0, 140)
    g1 = gpu_forward(G, f)
    G.set_option("er_fwd_reg", 0)
    g0 = gpu_forward(G, f)
    assert np.array_equal(g1, g0)
    assert_parity(g1, oracle.Geometry(d).forward(f), f"er forward registers ne={ne}")


def test_er_forward_registers_non_uniform_energies():
    d = make_config(0, energy_resolving=1).desc()
    d.update(energy_kev=np.array([30.0, 33.0, 41.0, 55.0, 60.0, 80.0, 101.0, 119.0]))
    G = P.Geometry(d)
    f = rnd(G.f_shape, 0, 141)
    g1 = gpu_forward(G, f)
    G.set_option("er_fwd_reg", 0)
    assert np.array_equal(g1, gpu_forward(G, f))
    assert_parity(g1, oracle.Geometry(d).forward(f), "er forward registers, non-uniform energies")

