"""Host-side behaviour of the drop-in API that needs no GPU.

Mirrors the reference's validation tests (test_grids.py:123-250) against this
package's GridProblem, and checks that the product path fails loudly -- never
silently computes on the CPU -- when no CUDA device is present.
"""

import numpy as np
import pytest

from paper_1511_04292_b200 import grids as G
from paper_1511_04292_b200.engine import constant_value


def line_problem(bc, n=4):
    u = np.zeros(n + 2)
    u[1:-1] = 10.0 * (1.0 + np.arange(n))
    return G.GridProblem(spacing=(1.0,), u=u, source=np.zeros(n),
                         center=np.full(n, 2.0), lower=(np.full(n, -1.0),),
                         upper=(np.full(n, -1.0),), bc=(bc,))


def test_boundary_rules():
    with pytest.raises(ValueError, match="boundary kind"):
        G.BoundaryRule("absorbing")
    with pytest.raises(ValueError, match="values"):
        G.BoundaryRule("face_dirichlet")
    with pytest.raises(ValueError, match="periodic"):
        line_problem((G.PERIODIC, G.MIRROR))
    p = line_problem((G.MIRROR, G.MIRROR))
    assert p.u[0] == p.u[1] and p.u[-1] == p.u[-2]
    p = line_problem((G.PERIODIC, G.PERIODIC))
    assert p.u[0] == p.u[-2] and p.u[-1] == p.u[1]
    p = line_problem((G.face_dirichlet(7.0), G.face_dirichlet(-1.0)))
    assert p.u[0] == 2 * 7.0 - p.u[1] and p.u[-1] == 2 * (-1.0) - p.u[-2]
    p = line_problem((G.FIXED, G.FIXED))
    p.u[0], p.u[-1] = 123.0, 456.0
    p.refresh_ghosts()
    assert p.u[0] == 123.0 and p.u[-1] == 456.0


def _kw(shape, **over):
    one = np.ones(shape)
    kw = dict(spacing=(1.0,) * len(shape), u=np.zeros(tuple(s + 2 for s in shape)),
              source=np.zeros(shape), center=one, lower=(one,) * len(shape),
              upper=(one,) * len(shape), bc=((G.FIXED, G.FIXED),) * len(shape))
    kw.update(over)
    return kw


@pytest.mark.parametrize("over,match", [
    (dict(u=np.zeros(4)), "ghost"),
    (dict(spacing=(1.0, 1.0)), "spacing"),
    (dict(lower=(np.ones(5),)), "neighbor"),
    (dict(center=np.array([1.0, 1.0, 0.0, 1.0])), "center"),
    (dict(mask=np.ones(5, dtype=bool)), "mask"),
])
def test_problem_validation(over, match):
    with pytest.raises(ValueError, match=match):
        G.GridProblem(**_kw((4,), **over))


def test_four_dimensional_rejected():
    with pytest.raises(ValueError, match="dimensional"):
        G.GridProblem(**_kw((3, 3, 3, 3)))


def test_zero_center_allowed_under_mask():
    c = np.ones(4)
    c[0] = 0.0
    p = G.GridProblem(**_kw((4,), center=c, mask=np.array([False, True, True, True])))
    assert p.shape == (4,)


def test_residual_history_csv(tmp_path):
    h = G.ResidualHistory(residual_inf=np.array([1.0, 0.5]),
                          true_residual_inf=np.array([2.0, 1.0]),
                          seconds=np.array([0.1, 0.2]), tolerance=1e-3,
                          converged=False)
    path = tmp_path / "h.csv"
    h.to_csv(path)
    lines = path.read_text().splitlines()
    assert lines[0] == "iteration,residual_inf,wall_seconds"
    assert lines[1] == "1,1,0.100000" and len(lines) == 3
    h.to_csv(path, timing=False)
    assert path.read_text().endswith(",0.000000\n")


def test_constant_detection_is_bitwise():
    assert constant_value(np.broadcast_to(3.5, (4, 4))) == 3.5
    a = np.full((3, 3), 2.0)
    assert constant_value(a) == 2.0
    a[1, 1] = -0.0 + 2.0 * (1 + 2 ** -52)
    assert constant_value(a) is None
    z = np.zeros((2, 2))
    z[0, 0] = -0.0
    assert constant_value(z) is None  # -0.0 and +0.0 differ in bits


def test_argument_errors_precede_device_use():
    p = G.GridProblem(**_kw((4, 4)))
    with pytest.raises(ValueError, match="traversal"):
        G.weighted_jacobi_sweep(p, 1.0, traversal="up")
    with pytest.raises(ValueError, match="SOR"):
        G.sor_solve(p, 2.5, 1e-6)


def test_unsupported_features_raise():
    q = G.GridProblem(**_kw((4, 4), bc=((G.MIRROR, G.MIRROR),) * 2))

    def computing_hook(u):
        u[0] = 2.0 * u[1] - u[2]

    q.post_sweep = computing_hook
    with pytest.raises(NotImplementedError):
        G.jacobi_solve(q, 1e-6)
    with pytest.raises(NotImplementedError):
        G.gauss_seidel_solve(q, 1e-6)


def test_no_cpu_fallback_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present; the GPU tests cover the device path")
    p = G.GridProblem(**_kw((8, 8)))
    with pytest.raises(RuntimeError, match="CUDA"):
        G.jacobi_solve(p, 1e-6)
    line = G.GridProblem(**_kw((4,)))  # 1-D grids are on the GPU path too (grids._LineGrid)
    with pytest.raises(RuntimeError, match="CUDA"):
        G.srj_solve(line, type("C", (), {"weight_sequence": np.ones(1)})(), 1e-6)


def test_post_sweep_gather_probe():
    """post_sweep hooks that copy values become a device gather (spherical
    tie_origin, problems.py:586-589); anything else is rejected."""
    shape = (6, 5, 7)

    def tie_origin(uu):
        uu[1] = uu[2]
        uu[0] = uu[2]

    dst, src = G.post_sweep_gather(tie_origin, shape)
    plane = 5 * 7
    assert np.array_equal(dst, np.arange(2 * plane))
    assert np.array_equal(src, 2 * plane + np.arange(2 * plane) % plane)

    def chain(uu):  # sequential copies -> simultaneous gather from originals
        uu[0] = uu[1]
        uu[1] = uu[2]

    d, s = G.post_sweep_gather(chain, (4, 3))
    assert np.array_equal(d, np.arange(6)) and np.array_equal(s, np.arange(3, 9))
    x = np.random.default_rng(0).standard_normal((4, 3))
    y = x.copy()
    chain(y)
    z = x.copy().reshape(-1)
    z[d] = x.reshape(-1)[s]
    assert np.array_equal(z.reshape(4, 3), y)

    d, s = G.post_sweep_gather(lambda uu: None, (4, 3))
    assert d.size == 0 and s.size == 0

    for bad in (lambda uu: uu.__setitem__(0, 2.0 * uu[1]),
                lambda uu: uu.__setitem__(0, uu[1] + 1.0),
                lambda uu: uu.__setitem__(0, uu[1] if uu[1, 0] > 3 else uu[2]),
                lambda uu: (_ for _ in ()).throw(RuntimeError("boom"))):
        with pytest.raises(NotImplementedError):
            G.post_sweep_gather(bad, (4, 3))


def test_coef_class_detection():
    """engine.coef_class: SRJ_COEF_* bits, bit for bit (include/srj.h)."""
    from paper_1511_04292_b200.engine import coef_class

    rng = np.random.default_rng(0)
    full = rng.random((5, 7))
    assert coef_class(full) == 0
    assert coef_class(np.broadcast_to(rng.random(7), (5, 7))) == 1
    assert coef_class(np.broadcast_to(rng.random((5, 1)), (5, 7))) == 2
    assert coef_class(np.full((5, 7), 3.0)) == 3
    assert coef_class(np.full((5, 1), 3.0)) == 1  # a one-column row is not classed
    z = np.zeros((4, 3))
    z[2, 1] = -0.0  # -0.0 == 0.0 numerically but not bitwise
    assert coef_class(z) == 0
    three = np.broadcast_to(rng.random((4, 1, 1)), (4, 3, 6))
    assert coef_class(three) == 2
    assert coef_class(np.broadcast_to(rng.random((1, 3, 1)), (4, 3, 6))) == 3
