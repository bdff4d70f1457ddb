"""CPU tests of the host-side logic: geometry/topology bookkeeping, material
law, bench flop model, configs.  Known answers from the reference tests
(test_*.py in the reference suite) and SURVEY §8(d)."""

import numpy as np
import pytest

from paper_2501_07778_b200.material import MaterialModel, constitutive_matrix, lame_constants
from paper_2501_07778_b200.mesh import SubdomainMesh
from paper_2501_07778_b200.topology import DomainTopology

UNIT = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])


def test_mesh_basics_and_errors():
    m = SubdomainMesh(UNIT, 3, {"left": "clamped"}, {"right": (1.0, 0.0)})
    assert m.n_side == 8 and m.n_elem == 7
    assert m.tag("left") == "clamped" and m.tag("top") == "free"
    assert np.allclose(m.node_coords()[7, 7], [1.0, 1.0])
    assert np.allclose(m.element_corners(0, 0)[2], [1 / 7, 1 / 7])
    assert m.is_parallelogram()
    assert m.side_length("right") == pytest.approx(1.0)
    i, j = m.side_node_indices("top")
    assert np.array_equal(j, np.full(8, 7)) and np.array_equal(i, np.arange(8))
    with pytest.raises(ValueError):
        SubdomainMesh(UNIT[::-1], 2)
    with pytest.raises(ValueError):
        SubdomainMesh(UNIT, 0)
    with pytest.raises(ValueError):
        SubdomainMesh(UNIT, 2, {"middle": "clamped"})
    with pytest.raises(ValueError):
        SubdomainMesh(UNIT, 2, {"left": "glued"})
    trap = SubdomainMesh(np.array([[0, 0], [1.1, 0], [1.3, 1.2], [0, 0.9]]), 2)
    assert not trap.is_parallelogram()


def test_material_law():
    c = constitutive_matrix(1.0, 0.3, "plane-stress")
    f = 1.0 / (1 - 0.09)
    assert np.allclose(c, [[f, 0.3 * f, 0], [0.3 * f, f, 0], [0, 0, f * 0.35]])
    lam, mu = lame_constants(1.0, 0.3)
    c2 = MaterialModel(1.0, 0.3, "plane-strain").C
    assert np.allclose(c2[0, 0], lam + 2 * mu) and np.allclose(c2[2, 2], mu)
    with pytest.raises(ValueError):
        constitutive_matrix(-1.0, 0.3)
    with pytest.raises(ValueError):
        constitutive_matrix(1.0, 0.5, "plane-strain")
    with pytest.raises(ValueError):
        constitutive_matrix(1.0, 0.3, "3d")


def test_lshape_topology():
    meshes = [SubdomainMesh(UNIT, 2), SubdomainMesh(UNIT + [1.0, 0.0], 2), SubdomainMesh(UNIT + [0.0, 1.0], 2)]
    topo = DomainTopology.from_subdomains(meshes)
    assert topo.q == 3 and topo.d == 2
    assert len(topo.interfaces) == 2 and len(topo.point_interfaces) == 1
    rec = topo.interfaces[0]
    assert (rec.m, rec.side_m, rec.p, rec.side_p, rec.reversed) == (0, "right", 1, "left", False)
    pts = topo.all_tied_pairs()
    assert len(pts) == 4 + 4 + 1
    recs = topo.partner_records(1)
    assert [(k, fl) for k, _, fl in recs] == [("side", True), ("point", False)]
    with pytest.raises(ValueError):
        DomainTopology.from_subdomains(meshes, tie_overrides={(1, 2): (0.0, 0.5)})


def test_partial_tie_and_reversed_interface():
    a = SubdomainMesh(UNIT, 2)
    b = SubdomainMesh(np.array([[2.0, 1.0], [1.0, 1.0], [1.0, 0.0], [2.0, 0.0]]), 2)  # rotated 180 deg
    topo = DomainTopology.from_subdomains([a, b], tie_overrides={(0, 1): (0.0, 0.5)})
    rec = topo.interfaces[0]
    assert rec.reversed and rec.tie_hi == 0.5
    (im, jm), (ip, jp) = topo.tied_side_pairs(rec)
    assert len(im) == 2


def test_bench_flop_model_matches_survey():
    import bench

    # 16x128 rounding = 2154.8 GFLOP; 4x16 = 0.17 GFLOP
    r = 16 * 128
    assert bench.round_flops([1] + [r] * 23 + [1], bench.expected_ranks(r)) / 1e9 == pytest.approx(2154.8, rel=1e-4)
    assert bench.round_flops([1] + [64] * 23 + [1], bench.expected_ranks(64)) / 1e9 == pytest.approx(0.174, rel=1e-2)
    flops, byts = bench.matvec_cost(16, 128)
    assert byts / 1e9 == pytest.approx(1.482, rel=2e-3)
    A, x = bench.make_inputs(4, 16)
    assert len(A) == 24 and A[1].shape == (4, 2, 2, 4) and x[5].shape == (16, 2, 16)


def test_configs_specs():
    from paper_2501_07778_b200.configs import config

    meshes, mat, body, eps = config(1)
    assert meshes[0].d == 5 and meshes[0].n_side == 32 and body == (0.0, -1.0) and eps == 1e-8
    meshes, mat, body, eps = config(4)
    assert meshes[0].d == 10 and mat.modulus_field is not None and meshes[0].tractions == {"right": (1.0, 0.0)}
    assert mat.modulus_field(np.array(0.25), np.array(0.25)) == pytest.approx(1.5)
    meshes, mat, body, eps = config(5)
    assert len(meshes) == 3 and meshes[2].tag("top") == "clamped" and mat.mode == "plane-strain"


def _throughput_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    import bench

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        local_ms = 10.0 * (rank + 1)  # rank 1 is the slow replica
        out[rank] = bench.job_throughput(local_ms, 2, 1e9, dist, world, torch.device("cpu"))
    finally:
        dist.destroy_process_group()


def test_replica_throughput_max_over_ranks_gloo():
    """bench.py's N>1 path (replicas, max-over-ranks step time) with the gloo
    backend and world_size 2 on CPU."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_throughput_worker, args=(2, port, out), nprocs=2, join=True)
    for rank in range(2):
        ms, value = out[rank]
        assert ms == pytest.approx(10.0)  # max(10, 20) ms over 2 steps
        assert value == pytest.approx(2 * 1e9 / 10e-3 / 1e9)
