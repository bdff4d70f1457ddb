"""Bilinear element kernels: drop-in for ``qttfem.element`` (element.py:17-263).

The per-element value grids of all 16 corner pairs are produced by ONE
device launch (``qtt_element_grids``); the reference-shaped host functions
(``element_stiffness_block`` etc.) slice that result and copy it back.
Per-Gauss-point geometry coefficients (the affine Jacobian expansion,
element.py:111-150) are a handful of scalars computed here on the host.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .material import MaterialModel
from .mesh import SubdomainMesh

__all__ = [
    "CORNERS",
    "shape_functions",
    "quadrature_rule",
    "jacobian_expansion",
    "element_stiffness_block",
    "element_load_block",
    "stiffness_value_grids",
    "load_value_grid",
    "traction_load",
    "value_grids",
]

CORNERS = ((-1, -1), (1, -1), (1, 1), (-1, 1))


def shape_functions(xi, eta):
    """Values (4,) and gradients (4, 2) of the Q1 corner functions."""
    xi = np.asarray(xi, dtype=np.float64)
    eta = np.asarray(eta, dtype=np.float64)
    sx = np.array([c[0] for c in CORNERS], dtype=np.float64)
    sy = np.array([c[1] for c in CORNERS], dtype=np.float64)
    fx = 1 + np.multiply.outer(sx, xi)
    fy = 1 + np.multiply.outer(sy, eta)
    vals = fx * fy / 4
    grads = np.stack([sx.reshape((4,) + (1,) * xi.ndim) * fy / 4, sy.reshape((4,) + (1,) * eta.ndim) * fx / 4], axis=1)
    return vals, grads


def quadrature_rule(name: str):
    """1-D tensor-product factors on [-1, 1] (element.py:56-63)."""
    if name == "gauss2":
        g = 1.0 / np.sqrt(3.0)
        return np.array([-g, g]), np.array([1.0, 1.0])
    if name == "midpoint":
        return np.array([0.0]), np.array([2.0])
    raise ValueError(f"unknown quadrature rule {name!r}")


def _jac(corner_xy, xi, eta):
    return shape_functions(xi, eta)[1].T @ corner_xy


def _expansion(mesh, xi, eta):
    j00 = _jac(mesh.element_corners(0, 0), xi, eta)
    if mesh.n_elem > 1:
        return (j00, _jac(mesh.element_corners(1, 0), xi, eta) - j00,
                _jac(mesh.element_corners(0, 1), xi, eta) - j00)
    return j00, np.zeros((2, 2)), np.zeros((2, 2))


def jacobian_expansion(mesh: SubdomainMesh, element, xi: float, eta: float,
                       paper_determinant: bool = False):
    """J^(i,j), (dxi/dx, deta/dx, dxi/dy, deta/dy) and |J| of one element."""
    i, j = element
    ne = mesh.n_elem
    if not (0 <= i < ne and 0 <= j < ne):
        raise ValueError(f"element ({i},{j}) out of range")
    j00, d10, d01 = _expansion(mesh, xi, eta)
    jac = j00 + i * d10 + j * d01
    if paper_determinant:
        det = np.linalg.det(j00) + i * np.linalg.det(d10) + j * np.linalg.det(d01)
    else:
        det = jac[0, 0] * jac[1, 1] - jac[0, 1] * jac[1, 0]
    if det <= 0:
        raise ValueError(f"degenerate element ({i},{j}): |J| = {det}")
    (x_xi, y_xi), (x_eta, y_eta) = jac
    return jac, (y_eta / det, -y_xi / det, -x_eta / det, x_xi / det), det


def _gauss_points(quadrature):
    pts, wts = quadrature_rule(quadrature)
    return [(gx, gy, wx * wy) for gx, wx in zip(pts, wts) for gy, wy in zip(pts, wts)]


def _modulus_grid(mesh, material, gps, dev):
    fld = getattr(material, "modulus_field", None)
    if fld is None:
        return None
    ne = mesh.n_elem
    idx = torch.arange(ne, dtype=torch.float64, device=dev)
    c = torch.as_tensor(mesh.corners, dtype=torch.float64, device=dev)
    out = torch.empty((len(gps), ne, ne), dtype=torch.float64, device=dev)
    for q, (gx, gy, _) in enumerate(gps):
        s = ((idx + (1 + gx) / 2) / ne)[:, None]
        t = ((idx + (1 + gy) / 2) / ne)[None, :]
        w = [(1 - s) * (1 - t), s * (1 - t), s * t, (1 - s) * t]
        x = sum(wk * c[k, 0] for k, wk in enumerate(w))
        y = sum(wk * c[k, 1] for k, wk in enumerate(w))
        out[q] = fld(x, y)
    return out


def value_grids(mesh: SubdomainMesh, material: MaterialModel, quadrature: str = "gauss2",
                paper_determinant: bool = False, ordering: str = "zorder"):
    """Device grids K (64, 4^d) [pair a*4+b, component] and G (16, 4^d),
    zero padded to 2^d x 2^d, flattened in ``ordering``."""
    dev = _lib.device()
    gps = _gauss_points(quadrature)
    coef = np.zeros((len(gps), 25))
    for q, (gx, gy, w) in enumerate(gps):
        vals, grads = shape_functions(gx, gy)
        j00, d10, d01 = _expansion(mesh, gx, gy)
        coef[q, 0:4] = j00.ravel()
        coef[q, 4:8] = d10.ravel()
        coef[q, 8:12] = d01.ravel()
        coef[q, 12] = w
        coef[q, 13:21] = grads.ravel()
        coef[q, 21:25] = vals
    cmat = np.ascontiguousarray(material.C, dtype=np.float64)
    npos = 1 << (2 * mesh.d)
    kout = torch.empty((64, npos), dtype=torch.float64, device=dev)
    gout = torch.empty((16, npos), dtype=torch.float64, device=dev)
    mod = _modulus_grid(mesh, material, gps, dev)
    deg = ctypes.c_int32(0)
    coef_c = np.ascontiguousarray(coef)
    _lib.call(
        "qtt_element_grids", ctypes.c_int32(mesh.d), ctypes.c_int32(1 if ordering == "zorder" else 0),
        ctypes.c_int32(len(gps)), coef_c.ctypes.data_as(ctypes.c_void_p),
        cmat.ctypes.data_as(ctypes.c_void_p), ctypes.c_int32(1 if paper_determinant else 0),
        _lib.ptr(mod), _lib.ptr(kout), _lib.ptr(gout), ctypes.byref(deg), _lib.stream_handle(),
    )
    if deg.value:
        raise ValueError("degenerate element in subdomain grid")
    return kout, gout


def _corner_index(c) -> int:
    try:
        return CORNERS.index(tuple(c))
    except ValueError:
        raise ValueError(f"unknown reference corner {c!r}") from None


def _canonical_elem(vec: torch.Tensor, d: int) -> np.ndarray:
    n = 1 << d
    return vec.view(n, n).t()[: n - 1, : n - 1].cpu().numpy()  # [i, j]


def element_stiffness_block(mesh, material, c1, c2, quadrature="gauss2", paper_determinant=False):
    """Grid (ne, ne, 2, 2) of K_{c1,c2} (element.py:160-195)."""
    a, b = _corner_index(c1), _corner_index(c2)
    kout, _ = value_grids(mesh, material, quadrature, paper_determinant, "canonical")
    p = a * 4 + b
    ne = mesh.n_elem
    out = np.empty((ne, ne, 2, 2))
    for c in range(4):
        out[:, :, c // 2, c % 2] = _canonical_elem(kout[p * 4 + c], mesh.d)
    return out


def element_load_block(mesh, c1, c2, quadrature="gauss2", paper_determinant=False):
    """Grid of G_{c1,c2} = sum_g W Phi_c1 Phi_c2 |J| (element.py:198-212)."""
    a, b = _corner_index(c1), _corner_index(c2)
    _, gout = value_grids(mesh, MaterialModel(1.0, 0.0), quadrature, paper_determinant, "canonical")
    return _canonical_elem(gout[a * 4 + b], mesh.d)


def stiffness_value_grids(mesh, material, quadrature="gauss2", paper_determinant=False) -> dict:
    kout, _ = value_grids(mesh, material, quadrature, paper_determinant, "canonical")
    ne = mesh.n_elem
    out = {}
    for a in range(4):
        for b in range(4):
            g = np.empty((ne, ne, 2, 2))
            for c in range(4):
                g[:, :, c // 2, c % 2] = _canonical_elem(kout[(a * 4 + b) * 4 + c], mesh.d)
            out[(a, b)] = g
    return out


def load_value_grid(mesh, quadrature="gauss2", paper_determinant=False) -> dict:
    _, gout = value_grids(mesh, MaterialModel(1.0, 0.0), quadrature, paper_determinant, "canonical")
    return {(a, b): _canonical_elem(gout[a * 4 + b], mesh.d) for a in range(4) for b in range(4)}


def traction_load(mesh, side, traction) -> np.ndarray:
    """Consistent nodal forces t*h (t*h/2 at the ends) of a constant traction
    on one side, as an (n, n, 2) node grid (element.py:244-263)."""
    if side not in mesh.tractions and traction is None:
        raise ValueError(f"side {side!r} carries no traction")
    t = np.asarray(mesh.tractions[side] if traction is None else traction, dtype=np.float64)
    n = mesh.n_side
    h = mesh.side_length(side) / mesh.n_elem
    w = np.full(n, h)
    w[[0, -1]] = h / 2
    out = np.zeros((n, n, 2))
    si, sj = mesh.side_node_indices(side)
    out[si, sj] = w[:, None] * t[None, :]
    return out
