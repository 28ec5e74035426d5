"""Multi-GPU and determinism on the device.

* Two processes, one GPU each, NCCL communicator from a unique id: each rank
  runs its cell / penalty-point partition and the one all-reduce per epoch;
  the result must equal the single-rank run (tolerance: the all-reduce sums
  the per-rank fp64 partials in a different order) and the replicas must stay
  bitwise identical.  Needs >= 2 visible devices (skipped on the 1-GPU boxes
  this round runs on; the partition arithmetic itself is covered on CPU by
  tests/test_partition_gloo.py).
* Acceptance criterion 9 (proj/tests/acceptance_main.cpp:460-491): two runs
  of the forward-accuracy setup (forward_sine.json: 2x2 cells, T=225,
  Q=1,600, the split path), 1,000 steps, bitwise-identical loss histories;
  the same on the C5 gear (the fused tensor-core step).
"""
import os
import sys

import numpy as np
import pytest

from oracle import pyoracle as po
from tests.gpu_helpers import c1_spec, gpu_from_oracle

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))


def _n_devices():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _rank_worker(rank, world, uid, spec, epochs, q):
    from paper_2404_12063_b200 import gpu as G
    ob = po.OracleProblem(spec, double=False)
    g = gpu_from_oracle(ob, spec, device=rank, rank=rank, world_size=world)
    g.set_params(ob.init_params().astype(np.float32))
    g.attach_comm(uid, world, rank)
    parts, grad = g.loss_and_grad()
    rep = g.train(epochs, lr0=1e-3)
    q.put((rank, parts, grad, rep.records["total"].copy(), g.get_params()))
    g.close()


@pytest.mark.skipif(_n_devices() < 2, reason="needs >= 2 GPUs (this round's boxes have one)")
@pytest.mark.parametrize("case", ["c1", "gear576"])
def test_nccl_two_ranks_match_single_rank(case):
    import multiprocessing as mp
    from paper_2404_12063_b200 import gpu as G
    from tests.test_gpu_parity import gear_spec
    spec = c1_spec() if case == "c1" else gear_spec()
    epochs = 20
    uid = G.nccl_unique_id()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, 2, uid, spec, epochs, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # replicas bitwise identical: every rank applies Adam to the same reduced vector
    for k in range(4):
        assert np.array_equal(np.asarray(out[0][k]).view(np.uint8), np.asarray(out[1][k]).view(np.uint8)), k
    _, g1 = _make(spec)
    parts1, grad1 = g1.loss_and_grad()
    rep1 = g1.train(epochs, lr0=1e-3)
    parts2, grad2, tot2, par2 = out[0]
    assert np.all(np.abs(parts2 - parts1) <= 1e-6 * np.abs(parts1) + 1e-30)
    assert np.abs(grad2 - grad1).max() <= 1e-6 * np.abs(grad1).max()
    r = np.abs(tot2 - rep1.records["total"]) / np.abs(rep1.records["total"])
    assert r.max() < 1e-5
    assert np.abs(par2 - g1.get_params()).max() < 1e-5


def _history(g, p0, n):
    g.set_params(p0)
    rep = g.train(n, lr0=1e-3)
    assert rep.steps_run == n
    rec = rep.records
    return np.stack([rec["total"], rec["variational"], rec["boundary"], rec["sensor"]]).copy()


@pytest.mark.parametrize("case", ["forward_sine", "c5_gear"])
def test_thousand_step_history_bitwise_identical(case):
    """acceptance_main.cpp:460-491 on the device: two runs (two contexts,
    then the same context again) of 1,000 steps give bitwise-identical
    histories (deterministic reductions, no atomics on the value path)."""
    import parity_cases as pc
    spec = pc.CASES[case]()
    ob = po.OracleProblem(spec, double=False)
    p0 = ob.init_params().astype(np.float32)
    ga = gpu_from_oracle(ob, spec)
    h1 = _history(ga, p0, 1000)
    gb = gpu_from_oracle(ob, spec)
    h2 = _history(gb, p0, 1000)
    h3 = _history(ga, p0, 1000)
    assert np.array_equal(h1.view(np.uint64), h2.view(np.uint64))
    assert np.array_equal(h1.view(np.uint64), h3.view(np.uint64))
    assert np.array_equal(ga.get_params().view(np.uint32), gb.get_params().view(np.uint32))
    assert np.all(np.isfinite(h1)) and h1[0, -1] < h1[0, 0]


# ---- the epoch tail over peer memory (vpinn_gpu_attach_peers) ----
@pytest.mark.parametrize("layers", [(2, 30, 30, 30, 1), (2, 50, 50, 50, 1)])
def test_peer_exchange_single_rank_is_bitwise_the_plain_path(layers):
    """world = 1 through the peer kernel (its own mailbox): the rank sum of
    one rank is exact, so loss, gradient, a 50-epoch history and the final
    parameters are the plain path's bits."""
    spec = c1_spec(layers=layers)
    ob = po.OracleProblem(spec, double=False)
    p0 = ob.init_params().astype(np.float32)
    ga = gpu_from_oracle(ob, spec)
    gb = gpu_from_oracle(ob, spec)
    gb.attach_peers([gb.peer_handle()], 1, 0)
    for g in (ga, gb):
        g.set_params(p0)
    pa, grad_a = ga.loss_and_grad()
    pb, grad_b = gb.loss_and_grad()
    assert np.array_equal(np.asarray(pa).view(np.uint64), np.asarray(pb).view(np.uint64))
    assert np.array_equal(grad_a.view(np.uint32), grad_b.view(np.uint32))
    ha, hb = _history(ga, p0, 50), _history(gb, p0, 50)
    assert np.array_equal(ha.view(np.uint64), hb.view(np.uint64))
    assert np.array_equal(ga.get_params().view(np.uint32), gb.get_params().view(np.uint32))


def _make(spec, **kw):
    """(oracle, GPU context with the oracle's p0) for a weak- or strong-form spec."""
    if spec.strong:
        from tests.test_strong_form import make_strong_pair
        ob, g, _ = make_strong_pair(spec, **kw)
        return ob, g
    ob = po.OracleProblem(spec, double=False)
    g = gpu_from_oracle(ob, spec, **kw)
    g.set_params(ob.init_params().astype(np.float32))
    return ob, g


def _peer_worker(rank, world, spec, epochs, q_out, q_handles, q_in):
    try:
        ob, g = _make(spec, device=0, rank=rank, world_size=world)
        q_handles.put((rank, g.peer_handle()))
        handles = q_in.get(timeout=300)
        g.attach_peers(handles, world, rank)
        parts, grad = g.loss_and_grad()
        rep = g.train(epochs, lr0=1e-3)
        q_out.put((rank, parts, grad, rep.records["total"].copy(), g.get_params()))
        g.close()
    except Exception as ex:  # noqa: BLE001
        q_out.put((rank, repr(ex)))
        raise


@pytest.mark.parametrize("case", ["c1", "gear576", "strong_sensors", "split_path", "paper_net"])
def test_peer_exchange_two_ranks_match_single_rank(case):
    """Two processes (both on device 0, where CUDA IPC maps each other's
    mailbox; on an 8-GPU node the same protocol runs over NVLink), each with
    its partition: the one-kernel epoch tail (reduce, rows into every
    rank's mailbox, rank-ordered sum, Adam) gives bitwise-identical replicas
    and the single-rank result within the reordered-sum tolerance."""
    import multiprocessing as mp
    from tests.test_gpu_parity import gear_spec
    from tests.test_strong_form import strong_spec
    spec = {"c1": c1_spec, "gear576": gear_spec,
            # 5,301 parameters: more rows than the device holds warps at once
            # (the exchange's grid is capped, warps stride over the rows)
            "paper_net": lambda: c1_spec(layers=(2, 50, 50, 50, 1)),
            "split_path": lambda: po.ProblemSpec(*po.structured_mesh(3, 2), n_test_1d=6, n_quad_1d=20,
                                                 forcing="sin4pi_f", boundary_g="sin4pi_u", n_boundary=200,
                                                 layers=(2, 30, 30, 30, 1), seed=42),
            "strong_sensors": lambda: strong_spec(bx=0.7, by=-0.4, eps_source=1, scalars=(1.5,), n_sensors=21,
                                                  sensor_field="sin2pi_u")}[case]()
    epochs, world = 20, 2
    ctx = mp.get_context("spawn")
    q_out, q_handles = ctx.Queue(), ctx.Queue()
    q_in = [ctx.Queue() for _ in range(world)]
    procs = [ctx.Process(target=_peer_worker, args=(r, world, spec, epochs, q_out, q_handles, q_in[r]))
             for r in range(world)]
    for p in procs:
        p.start()
    hs = dict(q_handles.get(timeout=300) for _ in range(world))
    for r in range(world):
        q_in[r].put([hs[i] for i in range(world)])
    res = [q_out.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for r in res:
        assert len(r) == 5, r
    out = dict((r[0], r[1:]) for r in res)
    for p in procs:
        assert p.exitcode == 0
    for k in range(4):
        assert np.array_equal(np.asarray(out[0][k]).view(np.uint8), np.asarray(out[1][k]).view(np.uint8)), k
    _, g1 = _make(spec)
    parts1, grad1 = g1.loss_and_grad()
    rep1 = g1.train(epochs, lr0=1e-3)
    parts2, grad2, tot2, par2 = out[0]
    assert np.all(np.abs(parts2 - parts1) <= 1e-6 * np.abs(parts1) + 1e-30)
    # the partition regroups the fp32 per-CTA sums (1e-5 for the order-2
    # strong form, as test_strong_rank_partition_sums_to_whole)
    gtol = 1e-5 if spec.strong else 1e-6
    assert np.abs(grad2 - grad1).max() <= gtol * np.abs(grad1).max()
    r = np.abs(tot2 - rep1.records["total"]) / np.abs(rep1.records["total"])
    assert r.max() < 1e-5
    assert np.abs(par2 - g1.get_params()).max() < 1e-5
