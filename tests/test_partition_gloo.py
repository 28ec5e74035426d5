"""Multi-GPU decomposition on CPU: world_size-2 gloo ranks each evaluate the
objective and gradient of the partition vpinn_gpu_create assigns them
(oracle, fp64), all-reduce(sum) like the per-epoch NCCL all-reduce of the
device path, and must reproduce the single-rank result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import pyoracle as po
from paper_2404_12063_b200 import _capi


def _spec(strong=False):
    nodes, cells = po.structured_mesh(5, 3, skew=0.15, skew_seed=1234)
    return po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=3, n_quad_1d=4, forcing="sin2pi_f",
                          boundary_g="sin2pi_u", n_boundary=37, n_sensors=11, sensor_seed=7,
                          sensor_field="sin2pi_u", eps=0.7, bx=0.3, by=-0.2, layers=(2, 8, 8, 1), seed=3,
                          strong=strong)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q, strong=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ob = po.OracleProblem(_spec(strong), double=True)
    p0 = ob.init_params()
    e0, e1, b0, b1, s0, s1 = _capi.partition(ob.E, ob.n_bnd, ob.n_sen, rank, world)
    parts, grad = ob.loss_and_grad_part(p0, e0, e1, b0, b1, s0, s1)
    buf = torch.tensor(np.concatenate([parts, grad]), dtype=torch.float64)
    dist.all_reduce(buf)  # the device path's single per-epoch all-reduce
    ranges = torch.tensor([e0, e1, b0, b1, s0, s1], dtype=torch.int64)
    gathered = [torch.zeros_like(ranges) for _ in range(world)]
    dist.all_gather(gathered, ranges)
    if rank == 0:
        out_q.put((buf.numpy(), [g.tolist() for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,strong", [(2, False), (3, False), (2, True)])
def test_partitioned_objective_sums_to_single_rank(world, strong):
    """weak form, and the strong-form collocation objective (whose residual
    mean uses the global interior count on every rank)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, strong)) for r in range(world)]
    for p in procs:
        p.start()
    red, ranges = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ob = po.OracleProblem(_spec(strong), double=True)
    parts, grad = ob.loss_and_grad(ob.init_params())
    np.testing.assert_allclose(red[:4], parts, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(red[4:], grad, rtol=1e-10, atol=1e-12 * np.abs(grad).max())
    # the partition tiles every range exactly once, contiguously
    for lo, n in ((0, ob.E), (2, ob.n_bnd), (4, ob.n_sen)):
        assert ranges[0][lo] == 0 and ranges[-1][lo + 1] == n
        for a, b in zip(ranges, ranges[1:]):
            assert a[lo + 1] == b[lo]


def test_partition_edge_cases():
    # more ranks than cells / penalty points: empty but well-formed slices
    for world in (1, 2, 7, 16):
        cover = []
        for r in range(world):
            e0, e1, b0, b1, s0, s1 = _capi.partition(5, 3, 0, r, world)
            assert 0 <= e0 <= e1 <= 5 and 0 <= b0 <= b1 <= 3 and s0 == s1 == 0
            cover.append((e0, e1))
        assert cover[0][0] == 0 and cover[-1][1] == 5
        assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))


# ---- bench.attach_ranks: the cross-rank attachment at N > 1 (host plumbing) ----
class _FakeCtx:
    """Stands in for GpuStep: records which attachment the rank made."""

    def __init__(self, rank, fail_handle=False, fail_attach=False):
        self.rank, self.fail_handle, self.fail_attach = rank, fail_handle, fail_attach
        self.peers = None
        self.comm = None

    def peer_handle(self):
        if self.fail_handle:
            raise RuntimeError("no IPC")
        return bytes([self.rank]) * 64

    def attach_peers(self, handles, world, rank):
        if self.fail_attach:
            raise RuntimeError("cannot map a peer")
        self.peers = list(handles)

    def attach_comm(self, uid, world, rank):
        self.comm = uid


def _attach_worker(rank, world, port, out_q, fail_rank, mode):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    import paper_2404_12063_b200.gpu as G
    G.nccl_unique_id = lambda: b"U" * 128  # no NCCL on the CPU box: the fallback's id only
    g = _FakeCtx(rank, fail_handle=(mode == "handle" and rank == fail_rank),
                 fail_attach=(mode == "attach" and rank == fail_rank))
    bench.attach_ranks(g, dist, world, rank)
    out_q.put((rank, g.peers is not None, g.comm is not None, g.peers))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["ok", "handle", "attach"])
def test_attach_ranks_agrees_on_one_collective(mode):
    """Every rank gathers the peer handles in rank order and attaches them;
    when any rank cannot export or map (mode handle / attach on rank 1) all
    ranks take NCCL together -- a rank that failed still joins the gather, so
    nobody blocks."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_attach_worker, args=(r, world, port, q, 1, mode)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if mode == "ok":
        for r in range(world):
            assert res[r][0] and not res[r][1]
            assert res[r][2] == [bytes([i]) * 64 for i in range(world)]
    else:
        for r in range(world):
            assert res[r][1], (mode, r, res[r])  # NCCL attached on every rank
