"""BASELINE.json configs 1, 4 and 5 as geometry/material specs.

Config 1: unit square, d=5 (32x32 nodes: the reference supports 2^d nodes
per side only), clamped at x=0, body force (0,-1), plane stress E=1, nu=0.3.
Config 4: unit square, d=10, clamped at x=0, traction (1,0) on x=1,
plane stress nu=0.3, E(x,y) = 1 + 0.5 sin(2 pi x) sin(2 pi y).
Config 5: L-shape of three unit patches (UNIT, UNIT+[1,0], UNIT+[0,1]),
clamp pinned to the top edge of patch 2 (outer end of the vertical leg),
plane strain E=1, nu=0.3, body force (0,-1).
"""

from __future__ import annotations

import numpy as np

from .material import MaterialModel, config4_modulus
from .mesh import SubdomainMesh

UNIT = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
EPS = 1e-8


def config(idx: int, d: int | None = None):
    """(meshes, material, body_force, eps) of BASELINE config ``idx``."""
    if idx == 1:
        d = 5 if d is None else d
        return [SubdomainMesh(UNIT, d, {"left": "clamped"})], MaterialModel(1.0, 0.3, "plane-stress"), (0.0, -1.0), EPS
    if idx == 4:
        d = 10 if d is None else d
        mesh = SubdomainMesh(UNIT, d, {"left": "clamped"}, {"right": (1.0, 0.0)})
        mat = MaterialModel(1.0, 0.3, "plane-stress", modulus_field=config4_modulus)
        return [mesh], mat, (0.0, 0.0), EPS
    if idx == 40:
        # SURVEY's "config-4-like" probe: config 4 with a constant E = 1
        d = 10 if d is None else d
        mesh = SubdomainMesh(UNIT, d, {"left": "clamped"}, {"right": (1.0, 0.0)})
        return [mesh], MaterialModel(1.0, 0.3, "plane-stress"), (0.0, 0.0), EPS
    if idx == 5:
        d = 10 if d is None else d
        meshes = [
            SubdomainMesh(UNIT, d),
            SubdomainMesh(UNIT + [1.0, 0.0], d),
            SubdomainMesh(UNIT + [0.0, 1.0], d, {"top": "clamped"}),
        ]
        return meshes, MaterialModel(1.0, 0.3, "plane-strain"), (0.0, -1.0), EPS
    raise ValueError(f"no config {idx}")


def build_system(idx: int, d: int | None = None, timings: dict | None = None,
                 assembly_eps: float | None = None):
    """Assemble, couple and constrain config ``idx`` on the device.

    ``assembly_eps`` (default: the config's eps, as BASELINE states it) is the
    tolerance of the assembly / coupling / Dirichlet roundings only; the
    returned eps is always the config's solve tolerance.  On config 4 the
    assembly tolerance, not the solver, sets the forward error: an operator
    assembled at 1e-8 has an exact solution 3.4e-5 away from the conforming
    FEM solution (condition ~1e7), one assembled at 1e-12 is 4e-9 away
    (profiles/r02_c4_error_probe.log)."""
    import time

    import torch

    from .assembly import assemble_subdomain
    from .coupling import apply_dirichlet, concat_blocks
    from .topology import DomainTopology

    meshes, mat, body, eps = config(idx, d)
    solve_eps = eps
    if assembly_eps is not None:
        eps = assembly_eps
    t0 = time.perf_counter()
    systems = [assemble_subdomain(m, mat, "zorder", eps, body_force=body) for m in meshes]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    topo = DomainTopology.from_subdomains(meshes)
    gsys = concat_blocks(systems, topo, ordering="zorder", epsilon=eps)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    gsys = apply_dirichlet(gsys, epsilon=eps)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if timings is not None:
        timings.update(assembly_s=t1 - t0, concat_s=t2 - t1, dirichlet_s=t3 - t2)
    return gsys, solve_eps
