"""Value-level pins of the oracle's TVB limiter paths that only whole-limiter runs reach
(readings A14-A16): the reflective-wall ghost of the TVB stencil, the
component-wise branch below h_char, and Eq. modified_TVB inside the limiter pipeline.

Each pin is a property fixed by the mathematics of the construction, not a retyped formula:

* Wall ghost = mirror image.  A reflective wall is the symmetry line of the mirror-extended
  problem (P:355 reflecting walls; A7).  The TVB limiter on a mesh with a wall at x = 0 must give
  exactly what it gives on the doubled mesh [-1,1] x [0,1] (the half mesh plus its mirror image)
  for the mirror-symmetric state h(-x,y) = h, hu(-x,y) = -hu, hv(-x,y) = hv.  In the doubled mesh
  the element across x = 0 is the mirror element: its barycentre is b0 reflected in the edge and
  its mean carries the mirrored normal momentum.
* Component-wise branch (A14: mean depth below h_char).  Limiting the conserved variables
  component by component involves no eigenvectors, so the limited state cannot depend on g; the
  characteristic branch (c = sqrt(g hbar)) does.
* Eq. modified_TVB: the limited P1 height is >= h0 at every vertex ("to ensure the
  positivity of the fluid height at the vertices"), and where the fix acts the smallest vertex
  value is exactly h0 (theta solves min vertex = h0).
"""
import numpy as np
import pytest

import oracle
import swe_inputs as si

N = 2
NP = (N + 1) * (N + 2) // 2
VERTS = [0, N, NP - 1]  # Nodes2D indices of the vertices (-1,-1), (1,-1), (-1,1)


def _half_and_doubled(nx=8, ny=8):
    """Half mesh [0,1]^2 (wall at x = 0) and the doubled mesh: the half mesh plus its mirror image
    in x = 0, sharing the vertices on x = 0.  Elements 0..K-1 of the doubled mesh are the half mesh."""
    m = si.structured(nx, ny, 0.0, 1.0, 0.0, 1.0)
    on = m.vx == 0.0
    nv = len(m.vx)
    new = np.cumsum(~on) - 1 + nv
    mp = np.where(on, np.arange(nv), new)
    vx2 = np.concatenate([m.vx, -m.vx[~on]])
    vy2 = np.concatenate([m.vy, m.vy[~on]])
    et2 = np.concatenate([m.etov, mp[m.etov]]).astype(np.int32)
    return (m.vx, m.vy, m.etov), (vx2, vy2, et2)


def _mirror_fields(x, y):
    ax = np.abs(x)
    h = 1.0 + 0.3 * np.sign(np.sin(9 * ax + 5 * y)) + 0.1 * np.cos(13 * y)
    hu = 0.8 * x * (1.0 + np.sin(7 * y))  # odd in x
    hv = 0.3 + 0.2 * np.cos(11 * ax)      # even in x
    return h, hu, hv


def _limit(mesh, fields, g=9.81, **kw):
    vx, vy, et = mesh
    prm = dict(h0=1e-6, tvb_M=0.0)
    prm.update(kw)
    o = oracle.Oracle(vx, vy, et, np.zeros((len(et), NP)), N, g, **prm)
    x, y = o.nodes()
    st = fields(x, y)
    return o, st, o.limit(*st)


def test_tvb_wall_ghost_is_the_mirror_image():
    half, dbl = _half_and_doubled()
    oh, inh, outh = _limit(half, _mirror_fields)
    od, ind, outd = _limit(dbl, _mirror_fields)
    K = len(half[2])
    for f in range(3):
        assert np.array_equal(inh[f], ind[f][:K])  # same input on the shared half
    # elements with a wall face on x = 0, and the ones TVB actually replaced
    e2e, _ = oh.connectivity()
    vxe = half[0][half[2]]
    at_wall = (np.sum(vxe == 0.0, axis=1) >= 2) & np.any(e2e == np.arange(K)[:, None], axis=1)
    changed = np.any(outh[0] != inh[0], axis=1) | np.any(outh[1] != inh[1], axis=1)
    assert (at_wall & changed).sum() >= 6
    assert oh.info()["n_tvb"] > 0 and oh.info()["n_tvb_cw"] == 0  # characteristic branch
    scale = [np.abs(a).max() for a in inh]
    for f in range(3):
        assert np.abs(outh[f] - outd[f][:K]).max() <= 1e-14 * scale[f], f


def _shallow_fields(base):
    def fields(x, y):
        h = base * (1 + 0.9 * np.sin(9 * x + 7 * y)) + 0.5 * base * np.sign(np.sin(15 * x))
        h = np.maximum(h, 1.5e-3)
        hu = 0.05 * np.sign(np.sin(11 * y)) * h / base
        hv = 0.02 * np.cos(8 * x) * h / base
        return h, hu, hv
    return fields


def test_tvb_component_wise_below_h_char_does_not_depend_on_g():
    m = si.structured(8, 8, 0.0, 1.0, 0.0, 1.0)
    mesh = (m.vx, m.vy, m.etov)
    h0 = 1e-3  # h_char = 10 h0 = 1e-2 > every mean depth of the shallow state
    oa, ina, outa = _limit(mesh, _shallow_fields(0.004), g=9.81, h0=h0)
    ob, inb, outb = _limit(mesh, _shallow_fields(0.004), g=1.0, h0=h0)
    ia = oa.info()
    assert ia["n_tvb"] > 20 and ia["n_tvb_cw"] == ia["n_tvb"] and ia["n_pp"] == 0
    for f in range(3):
        assert np.array_equal(outa[f], outb[f])
    # the characteristic branch (mean depth above h_char) does depend on g
    oc, _, outc = _limit(mesh, _shallow_fields(0.02), g=9.81, h0=h0)
    od, _, outd = _limit(mesh, _shallow_fields(0.02), g=1.0, h0=h0)
    assert oc.info()["n_tvb"] > oc.info()["n_tvb_cw"]
    assert max(np.abs(outc[f] - outd[f]).max() for f in range(3)) > 1e-6


@pytest.mark.parametrize("base", [0.004, 0.02])
def test_modified_tvb_keeps_the_vertices_at_or_above_h0(base):
    """Eq. modified_TVB through the whole limiter (Alg. 3, then TVB, then the fix), component-wise
    (base 0.004) and characteristic (base 0.02) branches."""
    m = si.structured(8, 8, 0.0, 1.0, 0.0, 1.0)
    mesh = (m.vx, m.vy, m.etov)
    h0 = 1e-3
    o, st, out = _limit(mesh, _shallow_fields(base), h0=h0)
    op, _, outp = _limit(mesh, _shallow_fields(base), h0=h0, use_tvb=0)
    i = o.info()
    assert i["n_pp"] == 0 and i["n_dry"] == 0  # Alg. 3 leaves this state alone: TVB alone acts
    changed = np.zeros(len(out[0]), dtype=bool)
    for f in range(3):
        changed |= np.any(out[f] != outp[f], axis=1)
    assert changed.sum() == i["n_tvb"] > 0
    vmin = out[0][:, VERTS].min(axis=1)
    assert vmin[changed].min() >= h0 * (1 - 1e-13)
    at_h0 = changed & (np.abs(vmin - h0) <= 1e-13 * h0)
    assert i["n_posfix"] >= 3 and at_h0.sum() == i["n_posfix"]
    # mean of every field preserved by the whole limiter (the fix keeps avg(Delta))
    wm = oracle.refel(N)["wmean"]
    for f in range(3):
        assert np.abs(0.5 * out[f] @ wm - 0.5 * st[f] @ wm).max() <= 1e-15 * max(1.0, np.abs(st[f]).max())


def test_tvb_nu_accepts_smooth_monotone_data():
    """The Cockburn-Shu factor nu > 1 (A14: nu = 1.5) is what lets the minmod accept smooth data:
    for a monotone quadratic height at rest the own midpoint deviation and the neighbour differences
    differ by O(H^2), so with nu = 1.5 every element with three real neighbours keeps its polynomial,
    while with nu = 1 (plain minmod of the two) every one of them is limited."""
    m = si.structured(8, 8, 0.0, 1.0, 0.0, 1.0)
    mesh = (m.vx, m.vy, m.etov)

    def smooth(x, y):
        h = 1 + 0.3 * x + 0.2 * y + 0.1 * (x * x + 0.5 * y * y + 0.5 * x * y)
        return h, np.zeros_like(x), np.zeros_like(x)

    res = {}
    for nu in (0.0, 1.0):  # 0 selects the default nu = 1.5
        o, st, out = _limit(mesh, smooth, tvb_nu=nu)
        e2e, _ = o.connectivity()
        interior = np.all(e2e != np.arange(len(m.etov))[:, None], axis=1)
        changed = np.any(out[0] != st[0], axis=1)
        res[nu] = (changed & interior).sum(), interior.sum()
    assert res[0.0][0] == 0 and res[1.0][0] == res[1.0][1] > 50, res
