"""Run the REFERENCE AMEn solver (qttfem.solver.solve, solver.py:239-389) on a
BASELINE system on this host's CPU cores, logging every residual evaluation
(one per sweep) with its wall time and the current solution ranks.

Development container only (imports /root/reference):

    PYTHONPATH=/root/reference/pkg/src python tools/ref_solve_cpu.py CONFIG D [MAX_SECONDS]

CONFIG 4  = config 4 as specified (variable E): the system is assembled by
            the oracle (oracle/fem.py, the SURVEY §8(c) modulus extension the
            reference lacks) and handed to the reference solver as reference
            TTMatrix/TTVector objects;
CONFIG 40 = config-4 geometry with constant E, assembled by the reference.
The solver runs with SolverConfig(epsilon=1e-8, seed=0, local_solver="direct")
(the default "auto" diverges).  The log lines are the
evidence quoted in DESIGN.md §8 / BASELINE.md (profiles/r02_ref_solve_*.log).
"""
from __future__ import annotations

import os
import signal
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import qttfem.solver as RS  # noqa: E402
import qttfem.ttcore as RT  # noqa: E402

cfg_idx = int(sys.argv[1])
d = int(sys.argv[2])
limit = float(sys.argv[3]) if len(sys.argv) > 3 else 3600.0

t0 = time.perf_counter()
if cfg_idx == 4:
    from oracle import fem as F
    from paper_2501_07778_b200.configs import config
    from paper_2501_07778_b200.topology import DomainTopology

    meshes, mat, body, eps = config(4, d)
    systems = F.assemble_all(meshes, mat, "zorder", eps, body)
    K, f, mask, gamma = F.concat(systems, DomainTopology.from_subdomains(meshes), eps=eps)
    K, f = F.dirichlet(K, f, mask, gamma, eps=eps)
    K, f = RT.TTMatrix(K), RT.TTVector(f)
else:
    import qttfem.assembly as RA
    import qttfem.coupling as RC
    from qttfem.material import MaterialModel
    from qttfem.mesh import SubdomainMesh
    from qttfem.topology import DomainTopology

    unit = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    mesh = SubdomainMesh(unit, d, {"left": "clamped"}, {"right": (1.0, 0.0)})
    eps = 1e-8
    sysm = RA.assemble_subdomain(mesh, MaterialModel(1.0, 0.3, "plane-stress"), "zorder", eps)
    g = RC.apply_dirichlet(RC.concat_blocks([sysm], DomainTopology.from_subdomains([mesh]), epsilon=eps),
                           epsilon=eps)
    K, f = g.K, g.f
t1 = time.perf_counter()
print(f"# config {cfg_idx} d={d}: build {t1 - t0:.1f}s, K ranks {K.ranks}, cores {os.cpu_count()}", flush=True)

_orig = RS.residual
calls = [0]


def logged(Kx, u, fx, rounding_eps=None):
    r = _orig(Kx, u, fx, rounding_eps)
    calls[0] += 1
    print(f"residual call {calls[0]}: {r:.3e}  max rank {max(u.ranks)}  t {time.perf_counter() - t1:.1f}s",
          flush=True)
    return r


RS.residual = logged


def _timeout(*_):
    print(f"# stopped after {limit:.0f}s without convergence", flush=True)
    os._exit(3)


signal.signal(signal.SIGALRM, _timeout)
signal.alarm(int(limit))
out = RS.solve(K, f, RS.SolverConfig(epsilon=eps, seed=0, local_solver="direct"))
print(f"# done: converged {out.converged} sweeps {out.sweeps} residual {out.residual:.3e} "
      f"ranks {out.u.ranks} solve {time.perf_counter() - t1:.1f}s", flush=True)
