"""BASELINE.json config 4 features that the reference does not have
(no reference oracle -- checked against closed forms and
scipy): integral-w equidistributed placement and the natural cubic-spline
interface fill.  Host-side C++ behind the C-ABI, so these run on CPU."""
import numpy as np
import pytest
from scipy.interpolate import CubicSpline

from paper_1310_3435_b200 import sdd

UNIT = sdd.RectDomain(0, 1, 0, 1)


def test_equidistributed_equals_equispaced_for_uniform_weight():
    m = sdd.MonitorFunction.constant()
    lay = sdd.build_layout(sdd.GridSpec(UNIT, 65, 65), 2, 2)
    a = sdd.plan_interface_points("equidistributed", 31, m, lay)
    b = sdd.plan_interface_points("equispaced", 31, m, lay)
    assert a.stochastic == b.stochastic


def test_equidistributed_places_nodes_by_integral_of_w():
    m = sdd.MonitorFunction.two_bump()
    spec = sdd.GridSpec(UNIT, 513, 513)
    lay = sdd.build_layout(spec, 4, 4)
    plan = sdd.plan_interface_points("equidistributed", 32, m, lay)
    assert len(plan.stochastic) == 6
    x = np.arange(513) / 512
    for ln, nodes in zip(lay.lines, plan.stochastic):
        assert 25 <= len(nodes) <= 32 and nodes == sorted(set(nodes))
        assert nodes[0] >= 1 and nodes[-1] <= 511
        # w along the line, trapezoid integral: nodes sit at equal shares within one cell
        if ln.vertical:
            w = 1 + 15 * np.exp(-100 * ((x[ln.fixed_index] - .3) ** 2 + (x - .3) ** 2)) + \
                15 * np.exp(-100 * ((x[ln.fixed_index] - .7) ** 2 + (x - .6) ** 2))
        else:
            w = 1 + 15 * np.exp(-100 * ((x - .3) ** 2 + (x[ln.fixed_index] - .3) ** 2)) + \
                15 * np.exp(-100 * ((x - .7) ** 2 + (x[ln.fixed_index] - .6) ** 2))
        cum = np.concatenate([[0], np.cumsum(0.5 * (w[1:] + w[:-1]))])
        share = cum[-1] / 33
        for j, p in enumerate(nodes):
            k = round(cum[p] / share)
            assert abs(cum[p] - k * share) <= 0.5 * (cum[p + 1] - cum[p - 1]) + 1e-12


def _fake(px, py, pid, f):
    out = np.zeros(len(px), sdd.ESTIMATE_DTYPE)
    out["xi"] = f(px, py)
    out["eta"] = f(py, px)
    out["walks"] = 1
    return out


def test_spline_fill_matches_scipy_natural_spline():
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 129, 129)
    lay = sdd.build_layout(spec, 2, 2)
    bd = sdd.make_boundary_data(m, spec, sdd.BC_IDENTITY)
    plan = sdd.plan_interface_points("equispaced", 9, m, lay)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    f = lambda a, b: np.sin(3 * a) * 0.3 + a + 0.1 * b
    est = _fake(px, py, pid, f)
    lin = sdd.fill_interfaces(m, lay, plan, bd, est, interp="linear")
    spl = sdd.fill_interfaces(m, lay, plan, bd, est, interp="spline")
    # vertical line (first): knots = endpoints + MC nodes
    knots = [0] + plan.stochastic[0] + [128]
    vals = spl.xi[0][knots]
    assert np.array_equal(vals, lin.xi[0][knots])          # knots are kept
    ref = CubicSpline(knots, vals, bc_type="natural")(np.arange(129))
    assert np.max(np.abs(spl.xi[0] - ref)) <= 1e-12
    assert np.max(np.abs(spl.xi[0] - lin.xi[0])) > 1e-6     # and it differs from linear


def test_spline_fill_reproduces_linear_data_exactly():
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 65, 65)
    lay = sdd.build_layout(spec, 2, 2)
    bd = sdd.make_boundary_data(m, spec, sdd.BC_IDENTITY)
    plan = sdd.plan_interface_points("equispaced", 7, m, lay)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    spl = sdd.fill_interfaces(m, lay, plan, bd, _fake(px, py, pid, lambda a, b: a), interp="spline")
    assert np.max(np.abs(spl.xi[1] - np.arange(65) / 64)) <= 1e-14   # horizontal line: xi = x


def test_unknown_interp_rejected():
    m = sdd.MonitorFunction.ring()
    spec = sdd.GridSpec(UNIT, 33, 33)
    lay = sdd.build_layout(spec, 2, 2)
    bd = sdd.make_boundary_data(m, spec)
    plan = sdd.plan_interface_points("equispaced", 3, m, lay)
    px, py, pid = sdd.interface_nodes(m, lay, plan)
    with pytest.raises(sdd.ValidationError):
        sdd.fill_interfaces(m, lay, plan, bd, _fake(px, py, pid, lambda a, b: a), interp="cubic")


@pytest.mark.gpu
def test_laplacian_smooth_is_the_four_neighbour_average(refimpl):
    # sddg_laplacian_smooth (config 4's "5 Laplacian sweeps"):
    # Perona-Malik FTCS with c = 1 and dt = h^2/4 is the 4-neighbour average
    # (to the rounding of u + dt * lap u), boundary kept; and it equals the
    # reference's perona_malik with the same mapping bit for bit
    from oracle import bindings as B
    n = 65
    spec = sdd.GridSpec(UNIT, n, n)
    rng = np.random.default_rng(1)
    x = np.linspace(0, 1, n)
    X, Y = np.meshgrid(x, x)
    xi = (X + 0.01 * rng.standard_normal((n, n)) * (X > 0) * (X < 1) * (Y > 0) * (Y < 1)).ravel()
    eta = (Y + 0.01 * rng.standard_normal((n, n)) * (X > 0) * (X < 1) * (Y > 0) * (Y < 1)).ravel()
    a, b = sdd.laplacian_smooth(xi, eta, spec, 5)
    u = xi.reshape(n, n).copy()
    for _ in range(5):
        v = u.copy()
        v[1:-1, 1:-1] = 0.25 * (u[1:-1, 2:] + u[1:-1, :-2] + u[2:, 1:-1] + u[:-2, 1:-1])
        u = v
    assert np.max(np.abs(a.reshape(n, n) - u)) < 1e-15
    assert np.array_equal(a.reshape(n, n)[0], xi.reshape(n, n)[0])
    rx, ry = refimpl.perona_malik(xi, eta, n, n, B.Domain(0, 1, 0, 1), 1e150, (1 / 64) ** 2 / 4, 5)
    assert np.array_equal(a, rx) and np.array_equal(b, ry)
