"""BASELINE.json's literal SDE dX = grad(w) dt + sqrt(2 w) dW as an opt-in
walk form (SDDG_FORM_LITERAL).  Its generator div(w grad) is
the reference's (1/w) div(w grad) times w: a time change, so the harmonic
functions and the exit law -- hence the estimates -- are the same, while
walks take fewer steps where w > 1.  No reference implementation exists, so
the check is statistical against the reference form: 4 combined standard
errors per node and field, exceedances against the null expectation and
chi^2/dof.  The literal form's step has standard deviation
sqrt(2 w dt): in the shock layer (w up to 21, width 0.02) it needs a step
about w_max times smaller for the same discretisation error, which the
shock case uses (at the reference form's dt the literal walks jump the layer
and the estimates are biased by many standard errors)."""
import math

import numpy as np
import pytest

from paper_1310_3435_b200 import sdd

pytestmark = pytest.mark.gpu
UNIT = sdd.RectDomain(0, 1, 0, 1)


def _z(a, b):
    z = []
    for f, s in (("xi", "se_xi"), ("eta", "se_eta")):
        se = np.hypot(a[s], b[s])
        ok = se > 0
        z.append((a[f][ok] - b[f][ok]) / se[ok])
    return np.concatenate(z)


@pytest.mark.parametrize("kind,n,s,dt,dt_lit,walks", [("ring", 65, 2, 5e-5, 5e-5, 20_000),
                                                       ("shock", 129, 4, 1e-5, 5e-7, 5_000),
                                                       ("two_bump", 129, 4, 5e-5, 5e-5, 20_000)])
def test_literal_form_has_the_reference_exit_law(ctx, kind, n, s, dt, dt_lit, walks):
    m = getattr(sdd.MonitorFunction, kind)(analytic=True)
    spec = sdd.GridSpec(UNIT, n, n)
    lay = sdd.build_layout(spec, s, s)
    px, py, pid = sdd.interface_nodes(m, lay, sdd.plan_interface_points("all", 0, m, lay))
    sel = np.linspace(0, len(px) - 1, 40).round().astype(int)
    pts, pid = np.stack([px[sel], py[sel]], 1), pid[sel]
    bd = sdd.make_boundary_data(m, spec)
    ref = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd, sdd.WalkConfig(scheme="linear", dt=dt, walks=walks,
                                                                      seed=1), ctx=ctx)
    zs = []
    for prec, seed in (("fp64", 2), ("fp32", 3)):
        lit = sdd.mc_estimate_batch(pts, pid, m, UNIT, bd,
                                    sdd.WalkConfig(scheme="linear", dt=dt_lit, walks=walks, seed=seed,
                                                   precision=prec, form="literal"), ctx=ctx)
        assert (lit["edge_hits"].sum(axis=1) == walks).all()
        # the time change: w >= 1 everywhere, so at equal dt literal walks are no longer
        if dt_lit == dt:
            assert lit["path_steps"].sum() < ref["path_steps"].sum()
        zs.append(_z(lit, ref))
    z = np.concatenate(zs)
    exceed = int(np.sum(np.abs(z) > 4))
    print(f"{kind}: {len(z)} z-values, |z|>4: {exceed} (null {len(z) * math.erfc(4 / math.sqrt(2)):.3f}), "
          f"chi2/dof {np.mean(z ** 2):.3f}")
    assert exceed <= 1
    assert abs(np.mean(z ** 2) - 1.0) <= 5 * math.sqrt(2.0 / len(z))


def test_literal_form_validation(ctx):
    bd = sdd.make_boundary_data(sdd.MonitorFunction.constant(), sdd.GridSpec(UNIT, 9, 9))
    with pytest.raises(sdd.ValidationError, match="BASELINE weights"):
        sdd.mc_estimate((0.5, 0.5), 0, sdd.MonitorFunction.constant(), UNIT, bd,
                        sdd.WalkConfig(scheme="linear", walks=4, form="literal"), ctx=ctx)
    with pytest.raises(sdd.ValidationError, match="linear scheme"):
        sdd.mc_estimate((0.5, 0.5), 0, sdd.MonitorFunction.ring(analytic=True), UNIT, bd,
                        sdd.WalkConfig(scheme="exponential", walks=4, form="literal"), ctx=ctx)
