"""Numpy restatement of the reference QTT assembly and coupling (oracle).

Follows /root/reference/pkg/src/qttfem/element.py, assembly.py and
coupling.py step for step (same term order, same epsilon splits, same
rounding points), on TT lists from ``oracle.tt``.  Geometry objects are
duck-typed (anything with the ``SubdomainMesh`` / ``DomainTopology``
attributes).  Config-4 extension: ``material.modulus_field`` (optional)
multiplies the stiffness integrand at each Gauss point by E(x_g, y_g)/E0,
(x_g, y_g) = mesh.map_point of the element's parametric Gauss point, and
forces the per-element branch.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

from __future__ import annotations

import numpy as np

from . import tt as O

CORNERS = ((-1, -1), (1, -1), (1, 1), (-1, 1))  # element.py:30
EXACT_EPS = 1e-13  # coupling.py:62
SIDE_AXIS = {"left": 0, "right": 0, "bottom": 1, "top": 1}
SIDE_POS = {"left": 0, "bottom": 0, "right": -1, "top": -1}


# ------------------------------------------------------------ element.py


def shape(xi, eta):
    """Q1 values (4,) and reference gradients (4, 2) (element.py:33-53)."""
    v = np.array([(1 - xi) * (1 - eta), (1 + xi) * (1 - eta), (1 + xi) * (1 + eta), (1 - xi) * (1 + eta)]) / 4
    g = np.array(
        [
            [-(1 - eta), -(1 - xi)],
            [(1 - eta), -(1 + xi)],
            [(1 + eta), (1 + xi)],
            [-(1 + eta), (1 - xi)],
        ]
    ) / 4
    return v, g


def gauss(rule):
    """element.py:56-63"""
    if rule == "gauss2":
        a = 1.0 / np.sqrt(3.0)
        return np.array([-a, a]), np.array([1.0, 1.0])
    if rule == "midpoint":
        return np.array([0.0]), np.array([2.0])
    raise ValueError(rule)


def _jac(corner_xy, xi, eta):
    return shape(xi, eta)[1].T @ corner_xy


def grid_jacobians(mesh, xi, eta, paper_det=False):
    """Affine expansion of J over the element grid (element.py:111-150)."""
    ne = mesh.n_elem
    j00 = _jac(mesh.element_corners(0, 0), xi, eta)
    if ne > 1:
        d10 = _jac(mesh.element_corners(1, 0), xi, eta) - j00
        d01 = _jac(mesh.element_corners(0, 1), xi, eta) - j00
    else:
        d10 = d01 = np.zeros((2, 2))
    ii, jj = np.meshgrid(np.arange(ne, dtype=float), np.arange(ne, dtype=float), indexing="ij")
    ent = {(a, b): j00[a, b] + ii * d10[a, b] + jj * d01[a, b] for a in (0, 1) for b in (0, 1)}
    if paper_det:
        det = np.linalg.det(j00) + ii * np.linalg.det(d10) + jj * np.linalg.det(d01)
    else:
        det = ent[0, 0] * ent[1, 1] - ent[0, 1] * ent[1, 0]
    if np.any(det <= 0):
        raise ValueError("degenerate element in subdomain grid")
    return ent[0, 0], ent[0, 1], ent[1, 0], ent[1, 1], det


def _modulus(mesh, material, gx, gy):
    fld = getattr(material, "modulus_field", None)
    if fld is None:
        return 1.0
    ne = mesh.n_elem
    ii, jj = np.meshgrid(np.arange(ne, dtype=float), np.arange(ne, dtype=float), indexing="ij")
    xy = mesh.map_point((ii + (1 + gx) / 2) / ne, (jj + (1 + gy) / 2) / ne)
    return np.asarray(fld(xy[..., 0], xy[..., 1]), dtype=float)


def stiffness_grid(mesh, material, a, b, rule="gauss2", paper_det=False):
    """(ne, ne, 2, 2) couplings of corners a, b (element.py:160-195)."""
    C = material.C
    pts, wts = gauss(rule)
    ne = mesh.n_elem
    out = np.zeros((ne, ne, 2, 2))
    for gx, wx in zip(pts, wts):
        for gy, wy in zip(pts, wts):
            grads = shape(gx, gy)[1]
            x_xi, y_xi, x_eta, y_eta, det = grid_jacobians(mesh, gx, gy, paper_det)
            w = wx * wy * det * _modulus(mesh, material, gx, gy)
            gX = [(grads[k, 0] * y_eta - grads[k, 1] * y_xi) / det for k in (a, b)]
            gY = [(-grads[k, 0] * x_eta + grads[k, 1] * x_xi) / det for k in (a, b)]
            out[..., 0, 0] += w * (C[0, 0] * gX[0] * gX[1] + C[2, 2] * gY[0] * gY[1])
            out[..., 0, 1] += w * (C[0, 1] * gX[0] * gY[1] + C[2, 2] * gY[0] * gX[1])
            out[..., 1, 0] += w * (C[0, 1] * gY[0] * gX[1] + C[2, 2] * gX[0] * gY[1])
            out[..., 1, 1] += w * (C[1, 1] * gY[0] * gY[1] + C[2, 2] * gX[0] * gX[1])
    return out


def load_grid(mesh, a, b, rule="gauss2", paper_det=False):
    """G_ab = sum_g W Phi_a Phi_b |J| (element.py:198-212)."""
    pts, wts = gauss(rule)
    out = np.zeros((mesh.n_elem, mesh.n_elem))
    for gx, wx in zip(pts, wts):
        for gy, wy in zip(pts, wts):
            v = shape(gx, gy)[0]
            out += wx * wy * v[a] * v[b] * grid_jacobians(mesh, gx, gy, paper_det)[4]
    return out


# ----------------------------------------------------------- assembly.py


def vec1d(values):
    values = np.asarray(values, float)
    if values.size == 2:
        return [values.reshape(1, 2, 1)]
    return O.decompose_vector(values, 0.0)


def ones1d(d):
    return [np.ones((1, 2, 1)) for _ in range(d)]


def unit1d(d, pos):
    out = []
    p = pos % (1 << d)
    for k in range(d):
        c = np.zeros((1, 2, 1))
        c[0, (p >> k) & 1, 0] = 1.0
        out.append(c)
    return out


def interval1d(d, lo, hi):
    """Sum of aligned dyadic block indicators (assembly.py:85-120)."""
    if lo > hi:
        return [np.zeros((1, 2, 1)) for _ in range(d)]
    acc = None
    a, b = lo, hi + 1
    while a < b:
        lev = 0
        while a % (1 << (lev + 1)) == 0 and a + (1 << (lev + 1)) <= b:
            lev += 1
        blk = []
        for k in range(d):
            if k < lev:
                blk.append(np.ones((1, 2, 1)))
            else:
                c = np.zeros((1, 2, 1))
                c[0, (a >> k) & 1, 0] = 1.0
                blk.append(c)
        acc = blk if acc is None else O.add(acc, blk)
        a += 1 << lev
    return acc


def compose2d(op_j, op_i, ordering):
    """assembly.py:131-141"""
    return O.kron(op_j, op_i) if ordering == "canonical" else O.zkron(op_j, op_i)


def grid_to_qtt(grid, ordering, eps=0.0):
    """assembly.py:144-158"""
    n = grid.shape[0]
    d = n.bit_length() - 1
    t = grid.reshape((2,) * (2 * d), order="F")
    if ordering == "zorder":
        t = t.transpose([ax for k in range(d) for ax in (k, d + k)])
    return O.decompose_vector(t.ravel(order="F"), eps, (2,) * (2 * d))


def shift1d(d, offset):
    """Rank-2 carry automaton (assembly.py:204-236)."""
    if d == 1:
        m = np.zeros((2, 2))
        m[0, offset] = 1.0
        return [m.reshape(1, 2, 2, 1)]
    I = np.eye(2)
    if offset == 1:
        s = np.array([[0.0, 1.0], [0.0, 0.0]])
        c = np.array([[0.0, 0.0], [1.0, 0.0]])
        first = np.stack([s, c], axis=-1).reshape(1, 2, 2, 2)
        mid = np.zeros((2, 2, 2, 2))
        mid[0, :, :, 0], mid[1, :, :, 0], mid[1, :, :, 1] = I, s, c
        last = np.zeros((2, 2, 2, 1))
        last[0, :, :, 0], last[1, :, :, 0] = I, s
    else:
        h = np.diag([0.0, 1.0])
        first = np.stack([I, h], axis=-1).reshape(1, 2, 2, 2)
        mid = np.zeros((2, 2, 2, 2))
        mid[0, :, :, 0], mid[1, :, :, 1] = I, h
        last = np.zeros((2, 2, 2, 1))
        last[0, :, :, 0], last[1, :, :, 0] = I, -h
    return [first] + [mid.copy() for _ in range(d - 2)] + [last]


def shift_operator(corner, d, ordering):
    """V_c (assembly.py:239-254)."""
    a = (corner[0] + 1) // 2
    b = (corner[1] + 1) // 2
    return compose2d(shift1d(d, b), shift1d(d, a), ordering)


def diag_grid(grid, ordering, eps=0.0):
    """assembly.py:257-267 (pads an (2^d - 1)^2 element grid)."""
    n = grid.shape[0]
    if n & (n - 1):
        d = n.bit_length()
        pad = np.zeros((1 << d, 1 << d))
        pad[:n, :n] = grid
        grid = pad
    return O.diag(grid_to_qtt(grid, ordering, eps))


def traction_vectors(mesh, side, tvec, ordering):
    """assembly.py:432-456"""
    d = mesh.d
    n = 1 << d
    h = mesh.side_length(side) / mesh.n_elem
    w = np.full(n, h)
    w[0] = w[-1] = h / 2
    sel = np.zeros(n)
    sel[0 if side in ("left", "bottom") else n - 1] = 1.0
    if side in ("left", "right"):
        v = compose2d(vec1d(w), vec1d(sel), ordering)
    else:
        v = compose2d(vec1d(sel), vec1d(w), ordering)
    return O.scale(v, tvec[0]), O.scale(v, tvec[1])


def assemble(mesh, material, ordering="zorder", eps=1e-12, rule="gauss2", body=(0.0, 0.0), paper_det=False):
    """Returns dict with kxx, kxy, kyx, kyy, fx, fy (tractions excluded)
    following assembly.py:321-429."""
    d = mesh.d
    ne = mesh.n_elem
    eacc = eps / 16.0
    V = [shift_operator(c, d, ordering) for c in CORNERS]
    const = mesh.is_parallelogram() and getattr(material, "modulus_field", None) is None
    pad = np.ones(1 << d)
    pad[-1] = 0.0
    ind = O.diag(compose2d(vec1d(pad), vec1d(pad), ordering))
    kz = [np.zeros((1, 2, 2, 1)) for _ in range(2 * d)]
    fz = [np.zeros((1, 2, 1)) for _ in range(2 * d)]
    K = [[kz, kz], [kz, kz]]
    F = [fz, fz]
    body = np.asarray(body, float)
    ones_nodes = [np.ones((1, 2, 1)) for _ in range(2 * d)]
    for a in range(4):
        for b in range(4):
            v1t = O.transpose(V[a])
            v2 = V[b]
            if const:
                coarse = _coarse(mesh)
                kv = stiffness_grid(coarse, material, a, b, rule, paper_det)[0, 0]
                gv = load_grid(coarse, a, b, rule, paper_det)[0, 0] / ne**2
                kd = {(p, q): O.scale(ind, kv[p, q]) for p in (0, 1) for q in (0, 1)}
                gd = O.scale(ind, gv)
            else:
                kg = stiffness_grid(mesh, material, a, b, rule, paper_det)
                gg = load_grid(mesh, a, b, rule, paper_det)
                kd = {(p, q): diag_grid(kg[:, :, p, q], ordering) for p in (0, 1) for q in (0, 1)}
                gd = diag_grid(gg, ordering)
            for p in (0, 1):
                for q in (0, 1):
                    term = O.matmat(O.matmat(v1t, kd[p, q]), v2)
                    K[p][q] = O.round_tt(O.add(K[p][q], term), eacc)
            if np.any(body != 0.0):
                gvec = O.matvec(O.matmat(O.matmat(v1t, gd), v2), ones_nodes)
                for p in (0, 1):
                    if body[p] != 0.0:
                        F[p] = O.round_tt(O.add(F[p], O.scale(gvec, body[p])), eacc)
    return {"kxx": K[0][0], "kxy": K[0][1], "kyx": K[1][0], "kyy": K[1][1], "fx": F[0], "fy": F[1]}


class _Coarse:
    """The d=1 copy of a mesh (same corners) used by the constant shortcut."""

    def __init__(self, mesh):
        self.corners = mesh.corners
        self.d = 1
        self.n_elem = 1
        self._m = mesh

    def element_corners(self, i, j):
        return self._m.map_point(np.array([0, 1, 1, 0.0]), np.array([0, 0, 1, 1.0]))

    def map_point(self, s, t):
        return self._m.map_point(s, t)


def _coarse(mesh):
    return _Coarse(mesh)


def with_tractions(sysd, mesh, ordering):
    """assembly.py:459-472"""
    out = dict(sysd)
    for side in sorted(mesh.tractions):
        tx, ty = traction_vectors(mesh, side, mesh.tractions[side], ordering)
        out["fx"] = O.round_tt(O.add(out["fx"], tx), 1e-14)
        out["fy"] = O.round_tt(O.add(out["fy"], ty), 1e-14)
    return out


def geometry_key(mesh, material, ordering, eps, rule, body, paper_det):
    """Translation-invariant key of the reference assembly cache (assembly.py:298-318)."""
    rel = np.round(mesh.corners - mesh.corners[0], 12)
    return (rel.tobytes(), mesh.d, material.youngs_modulus, material.poisson_ratio, material.mode,
            id(getattr(material, "modulus_field", None)), ordering, float(eps), rule,
            tuple(np.round(body, 15)), paper_det)


def assemble_all(meshes, material, ordering="zorder", eps=1e-12, body=(0.0, 0.0)):
    """Per-subdomain systems with the reference's cache sharing (cache=True):
    translated copies share the SAME block lists (identity grouping)."""
    cache = {}
    out = []
    for mesh in meshes:
        # the modulus field is position dependent: no sharing then
        key = geometry_key(mesh, material, ordering, eps, "gauss2", body, False)
        if getattr(material, "modulus_field", None) is not None:
            key = key + (mesh.corners.tobytes(),)
        if key not in cache:
            cache[key] = assemble(mesh, material, ordering, eps, "gauss2", body)
        base = cache[key]
        out.append(with_tractions(base, mesh, ordering) if mesh.tractions else dict(base))
    return out


# ----------------------------------------------------------- coupling.py


def _sel1d(d, pr, pc):
    n = 1 << d
    pr %= n
    pc %= n
    out = []
    for k in range(d):
        m = np.zeros((2, 2))
        m[(pr >> k) & 1, (pc >> k) & 1] = 1.0
        out.append(m.reshape(1, 2, 2, 1))
    return out


def _flip1d(d):
    return [np.array([[0.0, 1.0], [1.0, 0.0]]).reshape(1, 2, 2, 1) for _ in range(d)]


def _eye1d(d):
    return [np.eye(2).reshape(1, 2, 2, 1) for _ in range(d)]


def _tie_bounds(d, lo, hi):
    last = (1 << d) - 1
    return max(int(np.ceil(last * lo - 1e-9)), 0), min(int(np.floor(last * hi + 1e-9)), last)


def _tie_rows(d, rec, flipped):
    ka, kb = _tie_bounds(d, rec.tie_lo, rec.tie_hi)
    last = (1 << d) - 1
    if flipped and rec.reversed:
        ka, kb = last - kb, last - ka
    return interval1d(d, ka, kb)


def _side_pi(topo, rec, flipped, ordering):
    d = topo.d
    sm, sp = (rec.side_p, rec.side_m) if flipped else (rec.side_m, rec.side_p)
    along = O.matmat(O.diag(_tie_rows(d, rec, flipped)), _flip1d(d) if rec.reversed else _eye1d(d))
    cross = _sel1d(d, SIDE_POS[sm], SIDE_POS[sp])
    return compose2d(along, cross, ordering) if SIDE_AXIS[sm] == 0 else compose2d(cross, along, ordering)


def connectivity(topo, m, p, ordering="zorder"):
    """coupling.py:94-124"""
    d = topo.d
    terms = []
    for kind, rec, flipped in topo.partner_records(m):
        other = rec.m if flipped else rec.p
        if other != p:
            continue
        if kind == "side":
            terms.append(_side_pi(topo, rec, flipped, ordering))
        else:
            nm, npp = (rec.node_p, rec.node_m) if flipped else (rec.node_m, rec.node_p)
            terms.append(compose2d(_sel1d(d, nm[1], npp[1]), _sel1d(d, nm[0], npp[0]), ordering))
    if not terms:
        return [np.zeros((1, 2, 2, 1)) for _ in range(2 * d)]
    acc = terms[0]
    for t in terms[1:]:
        acc = O.add(acc, t)
    return acc


def multiplicity(topo, m, ordering="zorder"):
    """coupling.py:156-177"""
    d = topo.d
    acc = [np.zeros((1, 2, 1)) for _ in range(2 * d)]
    for kind, rec, flipped in topo.partner_records(m):
        if kind == "side":
            sm = rec.side_p if flipped else rec.side_m
            tie = _tie_rows(d, rec, flipped)
            sel = unit1d(d, SIDE_POS[sm])
            term = compose2d(tie, sel, ordering) if SIDE_AXIS[sm] == 0 else compose2d(sel, tie, ordering)
        else:
            node = rec.node_p if flipped else rec.node_m
            term = compose2d(unit1d(d, node[1]), unit1d(d, node[0]), ordering)
        acc = O.add(acc, term)
    return acc


def interface_forces(systems, topo, ordering="zorder"):
    """coupling.py:180-191"""
    out = []
    for m in range(topo.q):
        gx, gy = systems[m]["fx"], systems[m]["fy"]
        for _, rec, flipped in topo.partner_records(m):
            p = rec.m if flipped else rec.p
            pi = connectivity(topo, m, p, ordering)
            gx = O.round_tt(O.add(gx, O.matvec(pi, systems[p]["fx"])), EXACT_EPS)
            gy = O.round_tt(O.add(gy, O.matvec(pi, systems[p]["fy"])), EXACT_EPS)
        out.append((gx, gy))
    return out


def boundary_masks(mesh, d, ordering="zorder"):
    """coupling.py:202-226"""
    masks = []
    for comp in (0, 1):
        acc = [np.ones((1, 2, 1)) for _ in range(2 * d)]
        for side in ("left", "right", "bottom", "top"):
            tag = mesh.tag(side)
            if tag == "free" or (tag == "roller-x" and comp != 0) or (tag == "roller-y" and comp != 1):
                continue
            line = O.add(ones1d(d), O.scale(unit1d(d, SIDE_POS[side]), -1.0))
            term = compose2d(ones1d(d), line, ordering) if SIDE_AXIS[side] == 0 else compose2d(line, ones1d(d), ordering)
            acc = O.hadamard(acc, term)
        masks.append(acc)
    return masks


def default_gamma(systems, d):
    """Mean diagonal of Kxx, Kyy (coupling.py:299-309)."""
    tot, cnt = 0.0, 0
    for s in systems:
        for blk in (s["kxx"], s["kyy"]):
            g = np.ones((1, 1))
            for c in blk:
                g = g @ c[:, 0, 0, :] + g @ c[:, 1, 1, :]
            tot += float(g[0, 0])
            cnt += 4**d
    return tot / cnt


COMP = {
    (0, 0): np.array([[1.0, 0.0], [0.0, 0.0]]),
    (0, 1): np.array([[0.0, 1.0], [0.0, 0.0]]),
    (1, 0): np.array([[0.0, 0.0], [1.0, 0.0]]),
    (1, 1): np.array([[0.0, 0.0], [0.0, 1.0]]),
}


def _sub_qtt(pattern, s):
    if s == 0:
        return None
    return O.decompose_matrix(pattern, 0.0, (2,) * s, (2,) * s)


def _lift(block, sub, comp):
    cores = list(block) + (list(sub) if sub is not None else []) + [comp.reshape(1, 2, 2, 1)]
    return cores


def _lift_vec(vec, sub, comp):
    return list(vec) + (list(sub) if sub is not None else []) + [comp.reshape(1, 2, 1)]


def concat(systems, topo, gamma=None, ordering="zorder", eps=1e-12):
    """coupling.py:333-460 -> (K, f, mask, gamma).  ``systems`` come from
    assemble_all so identical (cached) blocks are the same list objects."""
    q, d = topo.q, topo.d
    if gamma is None:
        gamma = default_gamma(systems, d)
    s = 0 if q == 1 else int(np.ceil(np.log2(q)))
    qp = 1 << s

    def unit_pattern(m, p):
        e = np.zeros((qp, qp))
        e[m, p] = 1.0
        return e

    terms = []
    groups = {}
    names = {(0, 0): "kxx", (0, 1): "kxy", (1, 0): "kyx", (1, 1): "kyy"}
    for m, sy in enumerate(systems):
        for ab, nm in names.items():
            blk = sy[nm]
            key = (id(blk), ab)
            groups.setdefault(key, [np.zeros((qp, qp)), blk, ab])
            groups[key][0][m, m] = 1.0
    for pat, blk, ab in groups.values():
        terms.append((blk, pat, COMP[ab]))
    mgroups = {}
    for m in range(q):
        mk = multiplicity(topo, m, ordering)
        key = tuple((c.tobytes(), c.shape) for c in mk)
        mgroups.setdefault(key, [np.zeros((qp, qp)), mk])
        mgroups[key][0][m, m] = 1.0
    for pat, mk in mgroups.values():
        terms.append((O.scale(O.diag(mk), gamma), pat, np.eye(2)))
    for m in range(q):
        partners = sorted({(rec.m if fl else rec.p) for _, rec, fl in topo.partner_records(m)})
        for p in partners:
            pi = connectivity(topo, m, p, ordering)
            terms.append((O.scale(pi, -gamma), unit_pattern(m, p), np.eye(2)))
            for ab, nm in names.items():
                prod = O.round_tt(O.matmat(pi, systems[p][nm]), eps)
                terms.append((prod, unit_pattern(m, p), COMP[ab]))
    if qp > q:
        pad = np.zeros((qp, qp))
        pad[np.arange(q, qp), np.arange(q, qp)] = 1.0
        terms.append((O.scale(_eye1d(2 * d), gamma), pad, np.eye(2)))
    K = None
    eacc = eps / max(len(terms), 1)
    for blk, pat, comp in terms:
        lifted = _lift(blk, _sub_qtt(pat, s), comp)
        K = lifted if K is None else O.round_tt(O.add(K, lifted), eacc)
    loads = interface_forces(systems, topo, ordering)
    F = None
    for m, (gx, gy) in enumerate(loads):
        sub = unit1d(s, m) if s > 0 else None
        for comp, g in ((np.array([1.0, 0.0]), gx), (np.array([0.0, 1.0]), gy)):
            lifted = _lift_vec(g, sub, comp)
            F = lifted if F is None else O.round_tt(O.add(F, lifted), eacc)
    mask_groups = {}
    for m, sy in enumerate(systems):
        mx, my = boundary_masks(topo.subdomains[m], d, ordering)
        for ci, mv in enumerate((mx, my)):
            key = (ci,) + tuple(c.tobytes() for c in mv)
            mask_groups.setdefault(key, [np.zeros(qp), mv, ci])
            mask_groups[key][0][m] = 1.0
    tau = None
    for pat, mv, ci in mask_groups.values():
        sub = None
        if s > 0:
            for m in np.flatnonzero(pat):
                term = unit1d(s, int(m))
                sub = term if sub is None else O.add(sub, term)
        comp = np.zeros(2)
        comp[ci] = 1.0
        lifted = _lift_vec(mv, sub, comp)
        tau = lifted if tau is None else O.add(tau, lifted)
    return K, F, tau, gamma


def dirichlet(K, F, mask, gamma, gamma_bc=None, eps=1e-12):
    """K' = round(D K D) + gamma (I - D); f' = round(mask . f) (coupling.py:463-485)."""
    if gamma_bc is None:
        gamma_bc = gamma
    D = O.diag(mask)
    k = O.round_tt(O.matmat(D, O.matmat(K, D)), eps)
    ones = [np.ones((1, 2, 1)) for _ in range(len(mask))]
    comp = O.add(ones, O.scale(mask, -1.0))
    k = O.round_tt(O.add(k, O.scale(O.diag(comp), gamma_bc)), eps)
    f = O.round_tt(O.hadamard(mask, F), eps)
    return k, f
