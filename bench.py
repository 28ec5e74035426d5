#!/usr/bin/env python
"""FastVPINNs training-epoch benchmark on B200 (one JSON line on rank 0).

Workload (N=1 and every N): BASELINE config C5 — the ~14k-cell gear
(gen_fixtures.py recipe at n_r=16, n_t=887 -> 14,192 skewed quad cells),
gear_cd2d.json settings: cd2d eps=1, b=(0.1,0), gear_f, 5x5 test functions,
5x5 Gauss points (354,800 interior quadrature points), 800 boundary points,
MLP [2,30,30,30,1] tanh, Adam lr 1e-3, fp32.  A step = one full training
epoch (forward with tangents + Algorithm-3 contraction + penalty + reverse +
cross-rank gradient all-reduce + Adam), built through the product's C++ host
pipeline and run through the C-ABI.  Multi-GPU: cells and penalty points
are partitioned across ranks (strong scaling), one NCCL all-reduce per epoch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-sweep]

Beside the gear line, rank 0 at N=1 adds the C2 cell-count sweep (unit
square, 1..4,096 cells, "median ms/epoch vs cell count") and a C3 p/q sweep.

--impl reference times the reference algorithm's CPU implementation (the
plain-C++ oracle port: the reference itself cannot be built here, it needs
Eigen) on the same workload and metric, serial like the reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "median ms/epoch vs cell count; quad-pt evals/s; contraction HBM GB/s vs peak"
UNIT = "quad-pt evals/s"

GEAR_CFG = {
    "problem": {"pde": {"type": "cd2d", "eps": 1.0, "b": [0.1, 0.0]}, "forcing": "gear_f",
                "boundary_g": "zero", "n_boundary_points": 800},
    "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 5},
    "network": {"layers": [2, 30, 30, 30, 1]},
    "training": {"iterations": 1000, "learning_rate": 1e-3, "seed": 42, "precision": "single"},
}
GEAR_NR, GEAR_NT = 16, 887


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_source": "fallback B200_PROFILING.md"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        # NCCL init logs (rings / NVLS / nranks) for the driver's communicator check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,GRAPH")
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)  # host-side plumbing only
        pg = dist
    return world, rank, local, pg


COLLECTIVE = {"kind": None}


def attach_ranks(g, pg, world, rank):
    """Cross-rank plumbing of a context at N > 1: the peer-memory epoch tail
    (vpinn_gpu_attach_peers: every rank's mailbox mapped through CUDA IPC,
    reduce + rank sum + Adam in one kernel) -- the handles all-gathered over
    the gloo host group; NCCL (one all-reduce per epoch) if the peers cannot
    be mapped."""
    if world <= 1:
        return
    from paper_2404_12063_b200 import gpu as G
    import torch
    try:
        mine = g.peer_handle()
    except Exception:  # noqa: BLE001
        mine = None
    obj = [None] * world
    pg.all_gather_object(obj, mine)  # every rank joins the gather, also after a failure
    ok = 0
    if all(h is not None for h in obj):
        try:
            g.attach_peers(obj, world, rank)
            ok = 1
        except Exception:  # noqa: BLE001
            ok = 0
    t = torch.tensor([ok], dtype=torch.int32)
    pg.all_reduce(t, op=pg.ReduceOp.MIN)  # every rank takes the same path
    if int(t.item()) == 1:
        COLLECTIVE["kind"] = "peer memory (CUDA IPC over NVLink): one-kernel reduce + rank sum + Adam"
        return
    uid = bcast_bytes(pg, G.nccl_unique_id() if rank == 0 else b"", rank)
    g.attach_comm(uid, world, rank)
    COLLECTIVE["kind"] = "NCCL all-reduce (peer mapping unavailable)"


def bcast_bytes(pg, data: bytes, rank: int) -> bytes:
    if pg is None:
        return data
    obj = [data if rank == 0 else None]
    pg.broadcast_object_list(obj, src=0)
    return obj[0]


def allmax(pg, x: float) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


def build_problem():
    from paper_2404_12063_b200 import host
    mesh = host.Mesh.gear(GEAR_NR, GEAR_NT)
    return host.HostProblem(GEAR_CFG, mesh=mesh), mesh


def _gear_spec(strong=False):
    """The C5 gear problem as the oracle builds it; the mesh comes from the
    pure-Python generator (oracle/pyoracle.gear_mesh, the reference recipe,
    bit-identical to the product's), so the CPU legs load no product code."""
    from oracle import pyoracle as po
    nodes, cells = po.gear_mesh(GEAR_NR, GEAR_NT)
    return po.ProblemSpec(nodes=nodes, cells=cells, n_test_1d=5, n_quad_1d=5, forcing="gear_f",
                          boundary_g="zero", n_boundary=800, eps=1.0, bx=0.1, by=0.0,
                          layers=(2, 30, 30, 30, 1), seed=42, strong=strong)


def _pin_one_core():
    """Serial like the reference (proj/README.md:56-58): pin this process to
    one allowed core (taskset equivalent); returns (core, nproc)."""
    try:
        allowed = sorted(os.sched_getaffinity(0))
        core = allowed[-1]
        os.sched_setaffinity(0, {core})
        return core, len(allowed)
    except (AttributeError, OSError):
        return None, os.cpu_count()


def _unpin(prev):
    try:
        os.sched_setaffinity(0, prev)
    except (AttributeError, OSError):
        pass


def cpu_oracle_rate(max_seconds=25.0, strong=False):
    """The reference algorithm on the same gear problem, one pinned core:
    the TIMING build of the oracle port (the reference's -O3 -march=native
    flags, Eigen-style vectorised float tanh; oracle/Makefile 'native'),
    fp32, per-epoch seconds over a bounded sample."""
    from oracle import pyoracle as po
    try:
        prev = os.sched_getaffinity(0)
    except (AttributeError, OSError):
        prev = None
    core, nproc = _pin_one_core()
    try:
        ob = po.OracleProblem(_gear_spec(strong), double=False, timing_build=True)
        p0 = ob.init_params()
        first = ob.time_steps(p0, lr=1e-3, warmup=0, reps=1)[0]  # also the warm-up
        reps = int(max(2, min(8, (max_seconds - first) // max(first, 1e-3))))
        sec = ob.time_steps(p0, lr=1e-3, warmup=0, reps=reps)
    finally:
        if prev is not None:
            _unpin(prev)
    med = float(np.median(sec))
    return {"median_s": med, "reps": reps, "n_interior": ob.n_int, "cpu": cpu_model(), "core": core,
            "nproc": nproc}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, world, rank, pg):
    """--impl reference: the reference's CPU implementation on rank 0 only.

    The reference (proj/, header-only C++20 + Eigen) cannot be compiled here
    (Eigen 3.4 is absent), so the timed program is the plain-C++ restatement
    in oracle/ built with the reference's flags (-O3 -march=native, GNU
    dialect, Eigen-style vectorised float tanh: oracle/Makefile 'native'),
    serial and pinned to one core like the reference (proj/README.md:56-58).
    Same workload, metric, --steps and --warmup as the GPU arm; the protocol
    is trainer.hpp:153-172 (untimed warm-ups, then per-step seconds).  No
    product code is loaded: the gear comes from oracle/pyoracle.gear_mesh."""
    if rank != 0:
        return
    from oracle import pyoracle as po
    prev = os.sched_getaffinity(0) if hasattr(os, "sched_getaffinity") else None
    core, nproc = _pin_one_core()
    spec = _gear_spec()
    ob = po.OracleProblem(spec, double=False, timing_build=True)
    p0 = ob.init_params()
    warm, steps = args.warmup, args.steps
    sec = ob.time_steps(p0, lr=1e-3, warmup=warm, reps=steps)
    total = float(np.sum(sec))
    value = ob.n_int * steps / total
    # beside it (bounded): the checker build (libm tanh, no FMA contraction)
    # and the fp64 oracle, the reference's default precision (config.hpp:96)
    strict = po.OracleProblem(spec, double=False).time_steps(p0, lr=1e-3, warmup=0, reps=1)
    o64 = po.OracleProblem(spec, double=True, timing_build=True)
    f64 = o64.time_steps(o64.init_params(), lr=1e-3, warmup=0, reps=1)
    if prev is not None:
        _unpin(prev)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps,
        "median_ms_per_epoch": 1e3 * float(np.median(sec)), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic gear mesh (reference generator recipe, pure Python), seeded Glorot init",
        "config": {"workload": "C5 gear 14,192 cells (n_r=16,n_t=887), T=25, Q=25, cd2d eps=1 b=(0.1,0), "
                               "P_b=800, MLP [2,30,30,30,1] tanh, Adam lr 1e-3",
                   "sample": f"{steps} full epochs after {warm} warm-up epochs (same --steps/--warmup as the GPU arm)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "port",
                         "sample": f"{steps} full C5 epochs after {warm} warm-ups, one pinned core",
                         "cpu": cpu_model(), "nproc": nproc, "pinned_core": core,
                         "build": "oracle/Makefile native: -O3 -march=native (reference flags), Eigen-style float tanh",
                         "checker_build_s_per_epoch": float(strict[0]),
                         "fp64_s_per_epoch": float(f64[0]),
                         "note": "reference not buildable here (needs Eigen 3.4); plain-C++ restatement of its "
                                 "hot path, serial like the reference"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true",
                    help="skip the C2 cell-count and C3 p/q sweeps (a few seconds, rank 0 only)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world, rank, local, pg = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank, pg)
        return

    from paper_2404_12063_b200 import _capi, gpu as G
    hp, mesh = build_problem()
    E, Q, T = hp.E, hp.Q, hp.T
    device = local
    if world > 1:  # more ranks than devices (a functional check on a 1-GPU box): ranks share
        import torch
        device = local % max(1, torch.cuda.device_count())
    # ---- device context for this rank's partition ----
    step = G.GpuStep.from_problem(hp.view(device, rank, world), keepalive=hp)
    step.set_params(hp.init_params())
    attach_ranks(step, pg, world, rank)
    barrier(pg)

    import ctypes as C
    L = _capi.lib()
    # ---- warm-up (untimed), then K timed epochs, L2 flushed between epochs ----
    step.adam_reset()
    step.run_steps(args.warmup, 1e-3)
    step.synchronize()
    launches0 = step.launch_count()
    times = []
    with ClockSampler(device) as clk:
        barrier(pg)
        for k in range(args.steps):
            step.flush_l2()  # 256 MB write (> 126 MB L2) before, outside the timed epoch
            times.append(step.time_steps(1, 1e-3))
        step.synchronize()
        barrier(pg)
    launches = step.launch_count() - launches0
    # flush launches are not ours; time_steps counts only step kernels
    ms_total_local = float(np.sum(times))
    ms_total = allmax(pg, ms_total_local)
    ms_per_step = ms_total / args.steps
    P_total = E * Q if world == 1 else _global_interior(hp)
    value = P_total / (ms_per_step * 1e-3)

    # warm (L2-resident tensors, graph-replayed back to back) for reference
    warm_ms = step.time_steps(args.steps, 1e-3) / args.steps
    warm_ms = allmax(pg, warm_ms)

    # per-step device timestamps (median ms/epoch, the reference's statistic)
    rep = step.train(args.warmup + args.steps, lr0=1e-3)
    med_epoch_ms = 1e3 * float(np.median(rep.records["seconds"][args.warmup:]))
    med_epoch_ms = allmax(pg, med_epoch_ms)

    # ---- kernel shares and rooflines (rank 0 data is representative) ----
    ms_mlp, ms_red, ms_adam = step.profile_step(10)
    ffma = C.c_double()
    _capi.check(L.vpinn_gpu_measure_ffma_peak(device, C.byref(ffma)))
    ms_c, bytes_c = step.time_contract(20)
    kernel_name = step.step_kernel()
    pk = peaks()
    # algorithmic MLP flops per epoch of this rank: 33,180 per
    # interior point + 11,220 per boundary/sensor point at H=30
    n_int_local = hp.n_int // world if world > 1 else hp.n_int
    n_pen_local = (hp.n_bnd + hp.n_sen) // world if world > 1 else hp.n_bnd + hp.n_sen
    mlp_flops = 33180.0 * n_int_local + 11220.0 * n_pen_local
    mlp_tflops = mlp_flops / (ms_mlp * 1e-3) / 1e12
    contract_gbs = bytes_c / (ms_c * 1e-3) / 1e9

    # ---- end to end through the C-ABI with host buffers ----
    # (the timed context is released first: a user re-creating contexts gets
    # its device blocks from the library's block cache, as the e2e does here)
    step.close()
    # the end-to-end call chain three times (fresh contexts each), the median
    # reported: the first run in a process also pays one-time allocations
    def _median_e2e(pinned):
        runs = [_e2e(hp, device, rank, world, pg, args.steps, pinned) for _ in range(3)]
        r = sorted(runs, key=lambda r: r["seconds"])[1]
        r["runs_seconds"] = [x["seconds"] for x in runs]
        r["statistic"] = "median of 3 runs, each a fresh context"
        return r
    e2e_arrays = _median_e2e(True)
    e2e_pageable = _median_e2e(False)
    mesh_runs = [_e2e_from_mesh(mesh, device, rank, world, pg, args.steps) for _ in range(3)]
    e2e = sorted(mesh_runs, key=lambda r: r["seconds"])[1]
    e2e["runs_seconds"] = [x["seconds"] for x in mesh_runs]
    e2e["statistic"] = "median of 3 runs, each a fresh problem build and context"
    mf = _aux(_matrix_free, mesh, device, rank, world) if rank == 0 else None
    strong = _strong_form(mesh, device, rank, world, pg, args.steps, ms_per_step,
                          cpu=rank == 0 and world == 1 and not args.no_cpu_baseline)

    # ---- CPU baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            c = cpu_oracle_rate()
            cpu = {"value": c["n_interior"] / c["median_s"], "unit": UNIT, "cores": 1, "kind": "port",
                   "sample": f"median of {c['reps']} full C5 epochs (after 1 warm-up), fp32 oracle port, "
                             f"timing build (reference flags), pinned to core {c['core']} of {c['nproc']}",
                   "median_s_per_epoch": c["median_s"], "cpu": c["cpu"], "nproc": c["nproc"]}
        except Exception as ex:  # keep the GPU line even if the CPU leg fails
            cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {ex}"}

    aux = not args.no_sweep and rank == 0 and world == 1
    c4 = _aux(_c4_disk, device) if aux else None
    c4i = _aux(_c4_disk_spatial_inverse, device) if aux else None
    c5i = _aux(_c5_inverse, mesh, device) if aux else None
    c5p = _aux(_c5_paper, mesh, device) if aux else None
    sweep = _aux(_sweep, device) if aux else None
    sweep3 = _aux(_sweep_c3, device) if aux else None
    split = _aux(_c3_contraction, device, pk) if rank == 0 else None
    if rank != 0:
        return
    # the north star's "contraction HBM GB/s vs peak", kept inside roofline
    contraction = {"bound": "hbm",
                   "kernel": "contract_warp_kernel (standalone, warp per cell; compile-time 5x5/5x5 cell shape)",
                   "achieved": contract_gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                   "frac": contract_gbs / pk["hbm_gbs"],
                   "traffic": (_traffic("contract_warp") or {}).get("bytes"),
                   "bytes_per_launch": bytes_c, "ms_per_launch": ms_c,
                   "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic: gear mesh from the reference generator recipe, random-init (seeded Glorot) network",
        "config": {"workload": "C5 gear 14,192 cells (n_r=16,n_t=887), T=25, Q=25, cd2d eps=1 b=(0.1,0), "
                               "P_b=800, MLP [2,30,30,30,1] tanh, Adam lr 1e-3",
                   "cells": E, "n_test": T, "n_quad": Q, "interior_points": P_total,
                   "boundary_points": hp.n_bnd, "parallelism": f"cell-partitioned dp{world}",
                   "collective": COLLECTIVE["kind"],
                   "l2": "flushed (256 MB write) between timed epochs",
                   "warm_l2_ms_per_step": warm_ms, "median_ms_per_epoch": med_epoch_ms},
        "median_ms_per_epoch": med_epoch_ms,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "roofline": dict(_step_roofline(kernel_name, mlp_tflops, ffma.value, pk, ms_mlp / (ms_mlp + ms_red + ms_adam)),
                         contraction=contraction, contraction_split=split),
    }
    line.update({
        "kernel_ms": {"fused_step": ms_mlp, "reduce": ms_red, "adam": ms_adam},
        "e2e": e2e,
        "e2e_host_arrays": e2e_arrays,
        "e2e_pageable": e2e_pageable,
        "contraction_matrix_free": mf,
        "strong_form": strong,
        "cpu_baseline": cpu,
    })
    if sweep:
        line["sweep_c2"] = sweep
    if sweep3:
        line["sweep_c3"] = sweep3
    if c4:
        line["c4_disk"] = c4
    if c4i:
        line["c4_disk_spatial_inverse"] = c4i
    if c5i:
        line["c5_inverse"] = c5i
    if c5p:
        line["c5_paper_variant"] = c5p
    print(json.dumps(line), flush=True)


def _aux(fn, *args):
    """A rank-0 side measurement: its failure is reported in the line instead
    of costing the headline numbers."""
    try:
        return fn(*args)
    except Exception as ex:  # noqa: BLE001
        return {"error": f"{type(ex).__name__}: {ex}"}


def _traffic(kernel_prefix):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel
    from the round's committed ncu --set full capture (profiles/*traffic.json),
    or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                              "*traffic.json")), reverse=True):
        try:
            d = json.load(open(path))
        except Exception:
            continue
        for k, v in d.items():
            if k.startswith(kernel_prefix):
                return {"bytes": v, "source": os.path.relpath(path, os.path.dirname(os.path.abspath(__file__)))}
    return None


def _step_roofline(kernel_name, mlp_tflops, ffma_peak, pk, share):
    """Roofline of the dominant (fused step) kernel.  The tensor-core kernel
    computes every fp32 GEMM product as six bf16 tensor products (split-bf16,
    tc_utils.cuh), so its roofline peak is the measured bf16 tensor peak / 6
    in fp32-equivalent flop/s; the CUDA-core kernel's peak is the measured
    FFMA throughput.  'achieved' is always the ALGORITHMIC fp32 MLP flops
    (33,180 per interior point + 11,220 per penalty point) per
    launch over the launch time."""
    tc = kernel_name.startswith("tc_step") or kernel_name.startswith("tc2_step")
    tc2 = kernel_name.startswith("tc2_step")
    tr = _traffic("tc2_step" if tc2 else ("tc_step" if tc else "step_kernel"))
    if tc:
        # tc2: fp16 two-part split, 3 tensor products per fp32 product (fp16
        # runs at the bf16 rate); tc: bf16 three-part split, 6 products
        nprod = 3.0 if tc2 else 6.0
        peak = pk["bf16_tflops"] / nprod
        out = {"bound": "tensor", "kernel": kernel_name, "achieved": mlp_tflops, "peak": peak,
               "unit": "TFLOP/s", "frac": mlp_tflops / peak,
               "peak_source": f"MEASURED_PEAKS.json bf16_tflops (burst) / {nprod:.0f} tensor products per "
                              "fp32-faithful product",
               "fp32_ffma_equivalent": {"peak": ffma_peak, "frac": mlp_tflops / ffma_peak if ffma_peak else None,
                                        "peak_source": "FFMA microbenchmark measured in this run"}}
    else:
        out = {"bound": "fp32_fma", "kernel": kernel_name, "achieved": mlp_tflops, "peak": ffma_peak,
               "unit": "TFLOP/s", "frac": mlp_tflops / ffma_peak if ffma_peak else None,
               "peak_source": "FFMA microbenchmark measured in this run (no FP32 peak in MEASURED_PEAKS.json)"}
    out["traffic"] = tr["bytes"] if tr else None
    if tr:
        out["traffic_source"] = tr["source"]
    out["share_of_step"] = share
    out["algorithmic"] = "33,180 flop/interior pt + 11,220 flop/penalty pt (SURVEY 8d)"
    return out


def _global_interior(hp):
    return hp.E * hp.Q


_PINNED = {}


def _e2e(hp, device, rank, world, pg, steps, pinned=True):
    """Drop-in path: host ProblemAssembly arrays -> vpinn_gpu_create (H2D) ->
    train(K) -> parameters + history back to the host (D2H), wall-clocked.
    pinned: the input arrays sit in page-locked host memory (the contract's
    "inputs from pinned host memory"; copied there before the timed region)
    and are DMA'd from it directly; else they are the host assembly's own
    pageable arrays, staged through the library's pinned ring."""
    from paper_2404_12063_b200 import gpu as G
    view = hp.view(device, rank, world)
    keep = None
    if pinned:  # one page-locked copy per process, reused by the runs
        if id(hp) not in _PINNED:
            _PINNED[id(hp)] = G.pin_problem(view)
        view, keep = _PINNED[id(hp)]
    E, T, Q = hp.E, hp.T, hp.Q
    # bytes actually uploaded: 3 premultiplier tensors, forcing, float2 points,
    # float boundary targets, parameters
    h2d = 4 * (3 * E * T * Q + E * T) + 8 * (hp.n_int + hp.n_bnd + hp.n_sen) + 4 * hp.n_bnd + 4 * hp.n_params
    if world > 1:
        h2d //= world
    barrier(pg)
    t0 = time.perf_counter()
    g = G.GpuStep.from_problem(view, keepalive=(hp, keep))
    g.set_params(hp.init_params())
    attach_ranks(g, pg, world, rank)
    rep = g.train(steps, lr0=1e-3)
    params = g.get_params()
    t1 = time.perf_counter()
    g.close()
    dt = allmax(pg, t1 - t0)
    d2h = 4 * params.size + 7 * 8 * rep.steps_run
    return {"value": E * Q * steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d / steps),
            "d2h_bytes_per_step": int(d2h / steps), "seconds": dt,
            "inputs": "page-locked host memory" if pinned else "pageable host memory (staged)",
            "path": "vpinn_gpu_create(host arrays) + vpinn_gpu_train(K) + vpinn_gpu_get_params"}


def _e2e_from_mesh(mesh, device, rank, world, pg, steps):
    """The headline e2e: config + mesh in host memory -> trained parameters
    on the host, through the public API (HostProblem(device_assembly) ->
    vpinn_gpu_create with the assembly input -> train(K) -> get_params).
    The timed region covers the host problem build (config, rule and basis
    tables, boundary samples, Glorot init), the H2D copies of the mesh,
    tables, penalty points and parameters, the device assembly of the
    premultipliers (bit-identical to the host assembly:
    tests/test_device_assembly.py), K epochs and the D2H of the result.
    Beside it (e2e_host_arrays) the drop-in call with the host-assembled
    113 MB of premultipliers uploaded from page-locked memory."""
    from paper_2404_12063_b200 import gpu as G, host
    barrier(pg)
    t0 = time.perf_counter()
    dp = host.HostProblem(GEAR_CFG, mesh=mesh, device_assembly=True)
    g = G.GpuStep.from_problem(dp.view(device, rank, world), keepalive=dp)
    g.set_params(dp.init_params())
    attach_ranks(g, pg, world, rank)
    rep = g.train(steps, lr0=1e-3)
    params = g.get_params()
    t1 = time.perf_counter()
    g.close()
    dt = allmax(pg, t1 - t0)
    E, T, Q = dp.E, dp.T, dp.Q
    e_local = E // world if world > 1 else E
    # nodes (double2), cell node ids (int4), rule (3 Q doubles), basis tables
    # (3 T Q doubles) and their float copies for the matrix-free contraction,
    # penalty points (float2) and targets (float), parameters
    h2d = (16 * mesh.n_nodes + 16 * e_local + (8 + 4) * 3 * Q + (8 + 4) * 3 * T * Q
           + 12 * (dp.n_bnd + dp.n_sen) + 4 * dp.n_params)
    d2h = 4 * params.size + 7 * 8 * rep.steps_run
    return {"value": E * Q * steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d / steps),
            "d2h_bytes_per_step": int(d2h / steps), "seconds": dt,
            "inputs": "config + mesh (nodes, cells) in host memory",
            "path": "HostProblem(config, mesh, device_assembly) + vpinn_gpu_create(assembly input) + "
                    "vpinn_gpu_train(K) + vpinn_gpu_get_params"}


def _matrix_free(mesh, device, rank, world):
    """the matrix-free contraction (basis tables + per-cell
    geometry, contract_mf.cuh) on the same gear cells, L2 flushed per launch;
    a different algorithm from the paper's premultiplier tensors, reported
    beside the HBM-roofline contraction, not instead of it."""
    from paper_2404_12063_b200 import gpu as G, host
    dp = host.HostProblem(GEAR_CFG, mesh=mesh, device_assembly=True)
    g = G.GpuStep.from_problem(dp.view(device, rank, world), keepalive=dp)
    ms, nbytes = g.time_contract_matrix_free(20)
    g.close()
    return {"kernel": "contract_mf_kernel", "ms_per_launch": ms, "bytes_per_launch": nbytes,
            "achieved_GBs": nbytes / (ms * 1e-3) / 1e9,
            "note": "HBM bytes 14x below the premultiplier stream; shared-memory-load bound on CUDA cores"}


# mma.sync m16n8k8 TF32 issue rate measured on this pool's B200
# (tools/micro/mma_sync_rate.cu, profiles/r01_mma_sync_rate.txt)
MMA_SYNC_TF32_TFLOPS = 277.0


def _strong_form(mesh, device, rank, world, pg, steps, weak_ms, cpu=False):
    """the strong-form collocation baseline (the paper's
    PINN comparison) on the same gear workload: order-2 network at the
    354,800 interior quadrature points + the boundary penalty, one tcgen05
    step kernel (sf2_step_kernel.cuh) + the same reduce/Adam.  Device-timed
    epochs, L2 flushed between them, max over ranks."""
    import copy
    from paper_2404_12063_b200 import gpu as G, host
    cfg = copy.deepcopy(GEAR_CFG)
    cfg["discretization"]["form"] = "strong"
    hp = host.HostProblem(cfg, mesh=mesh)
    g = G.GpuStep.from_problem(hp.view(device, rank, world), keepalive=hp)
    g.set_params(hp.init_params())
    attach_ranks(g, pg, world, rank)
    g.adam_reset()
    g.run_steps(5, 1e-3)
    g.synchronize()
    barrier(pg)
    times = []
    for _ in range(max(5, min(steps, 30))):
        g.flush_l2()
        times.append(g.time_steps(1, 1e-3))
    ms = allmax(pg, float(np.median(times)))
    ms_k, ms_r, ms_a = g.profile_step(10)
    kernel = g.step_kernel()
    g.close()
    n_pts = (hp.n_int + hp.n_bnd + hp.n_sen) // max(1, world)
    # algorithmic: ~55,050 flop per point for [2,30,30,30,1] (5 streams x
    # (2 forward + 2 propagation + 2 weight-gradient) 30x30 products = 54,000
    # + the input / output layers)
    alg_tflops = n_pts * 55050.0 / (ms_k * 1e-3) / 1e12
    if kernel.startswith("sf2_step"):
        peak = peaks()["bf16_tflops"] / 3.0
        roof = {"bound": "tensor", "pipe": "tcgen05 kind::f16, fp16 two-part split (3 products per fp32 product)",
                "achieved": alg_tflops, "peak": peak, "unit": "TFLOP/s", "frac": alg_tflops / peak,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) / 3"}
    else:
        # executed: 1,440 m16n8k8 MMAs (3-pass TF32 split, widths padded to 32)
        # per 16-point tile
        exec_tflops = -(-n_pts // 16) * 1440 * 2 * 16 * 8 * 8 / (ms_k * 1e-3) / 1e12
        roof = {"bound": "tensor", "pipe": "mma.sync TF32 (legacy HMMA)", "achieved": exec_tflops,
                "peak": MMA_SYNC_TF32_TFLOPS, "unit": "TFLOP/s", "frac": exec_tflops / MMA_SYNC_TF32_TFLOPS,
                "algorithmic_tflops": alg_tflops, "peak_source": "tools/micro/mma_sync_rate.cu on this pool's B200"}
    return {"workload": "C5 gear, form=strong: PINN collocation residual at the interior quadrature points "
                        "+ boundary penalty, same network / points / Adam",
            "kernel": kernel, "ms_per_epoch": ms, "points_per_s": (hp.n_int + hp.n_bnd + hp.n_sen) / (ms * 1e-3),
            "strong_over_weak_epoch_time": ms / weak_ms if weak_ms else None,
            "kernel_ms": {"step": ms_k, "reduce": ms_r, "adam": ms_a},
            "roofline": roof,
            "l2": "flushed between timed epochs",
            "cpu_baseline": _strong_cpu(mesh) if cpu else None}


def _strong_cpu(mesh):
    """The reference's strong-form algorithm (oracle port, fp32, 1 core) on
    the same gear points: a bounded sample of full epochs."""
    try:
        c = cpu_oracle_rate(max_seconds=12.0, strong=True)
        return {"value": c["n_interior"] / c["median_s"], "unit": UNIT, "cores": 1, "kind": "port",
                "sample": f"median of {c['reps']} full strong-form gear epochs (after 1 warm-up), fp32 oracle port",
                "median_s_per_epoch": c["median_s"]}
    except Exception as ex:  # keep the GPU line even if the CPU leg fails
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "port", "sample": f"failed: {ex}"}


def _flushed_epoch_ms(hp, device, reps=20):
    from paper_2404_12063_b200 import gpu as G
    g = G.GpuStep.from_problem(hp.view(device), keepalive=hp)
    g.set_params(hp.init_params())
    g.adam_reset()
    g.run_steps(10, 1e-3)
    g.synchronize()
    times = []
    for _ in range(reps):
        g.flush_l2()
        times.append(g.time_steps(1, 1e-3))
    kernel = g.step_kernel()
    g.close()
    return float(np.median(times)), kernel


def _c5_inverse(mesh, device):
    """C5 inverse: the gear with a trainable scalar eps (init 2.0) and 50
    sensors (values from a named field, seed 7); device-timed, L2 flushed."""
    import copy
    from paper_2404_12063_b200 import host
    cfg = copy.deepcopy(GEAR_CFG)
    cfg["problem"]["exact_solution"] = "sin2pi_u"
    cfg["problem"]["sensors"] = {"count": 50, "seed": 7}
    cfg["network"]["eps_scalar_init"] = 2.0
    hp = host.HostProblem(cfg, mesh=mesh)
    ms, kernel = _flushed_epoch_ms(hp, device)
    return {"cells": hp.E, "sensors": hp.n_sen, "ms_per_epoch": ms, "kernel": kernel,
            "quad_pt_evals_per_s": hp.n_int / (ms * 1e-3), "l2": "flushed between timed epochs"}


def _c5_paper(mesh, device):
    """The paper's gear variant: T=16 (4x4), Q=25,
    6,096 boundary points, [2,50,50,50,1]; H = 50 runs on the tensor-core
    step in its 64-wide class (512 threads, 112-point tiles, one CTA per SM).
    Algorithmic MLP work at H = 50 (SURVEY 8d formula): 2 (18 H^2 + 13 H) =
    91,300 flop per interior point, 2 (6 H^2 + 7 H) = 30,700 per penalty
    point, over the whole (L2-flushed) epoch time."""
    import copy
    from paper_2404_12063_b200 import host
    cfg = copy.deepcopy(GEAR_CFG)
    cfg["discretization"]["n_test_per_dim"] = 4
    cfg["problem"]["n_boundary_points"] = 6096
    cfg["network"]["layers"] = [2, 50, 50, 50, 1]
    hp = host.HostProblem(cfg, mesh=mesh)
    ms, kernel = _flushed_epoch_ms(hp, device)
    flops = 91300.0 * hp.n_int + 30700.0 * (hp.n_bnd + hp.n_sen)
    tflops = flops / (ms * 1e-3) / 1e12
    peak = peaks()["bf16_tflops"] / 3.0
    return {"cells": hp.E, "n_test": hp.T, "n_quad": hp.Q, "boundary_points": hp.n_bnd, "layers": [2, 50, 50, 50, 1],
            "ms_per_epoch": ms, "kernel": kernel, "quad_pt_evals_per_s": hp.n_int / (ms * 1e-3),
            "mlp_tflops_algorithmic": tflops, "frac_of_bf16_over_3": tflops / peak,
            "l2": "flushed between timed epochs"}


def _c4_disk(device):
    """C4: convection-diffusion on the circular domain, 32x32 = 1,024 skewed
    cells with per-cell bilinear Jacobians, T=25, Q=100, b=(1,0), constant
    forcing; device-timed epochs, L2 flushed."""
    from paper_2404_12063_b200 import host
    cfg = {"problem": {"pde": {"type": "cd2d", "eps": 1.0, "b": [1.0, 0.0]}, "forcing": "one",
                       "boundary_g": "zero", "n_boundary_points": 400},
           "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
           "network": {"layers": [2, 30, 30, 30, 1]},
           "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    hp = host.HostProblem(cfg, mesh=host.Mesh.disk(32))
    ms, kernel = _flushed_epoch_ms(hp, device)
    return {"cells": hp.E, "n_test": hp.T, "n_quad": hp.Q, "ms_per_epoch": ms, "kernel": kernel,
            "quad_pt_evals_per_s": hp.n_int / (ms * 1e-3), "l2": "flushed between timed epochs"}


def _c4_disk_spatial_inverse(device):
    """The paper's space-dependent-coefficient inverse on
    C4's circular domain: 1,024 skewed cells, cd2d with b = (1, 0), the
    network's second output channel eps(x, y) = softplus(y1)
    (network.hpp:130-138, 477-483), 50 sensors; T = 25, Q = 100, constant
    forcing (the reference's field set has no f = 10; the cost is the same).
    Device-timed epochs, L2 flushed."""
    from paper_2404_12063_b200 import host
    cfg = {"problem": {"pde": {"type": "cd2d_variable_eps", "b": [1.0, 0.0]}, "forcing": "one",
                       "boundary_g": "zero", "exact_solution": "sinpi_u", "n_boundary_points": 400,
                       "sensors": {"count": 50, "seed": 7}},
           "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
           "network": {"layers": [2, 30, 30, 30, 2]},
           "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    hp = host.HostProblem(cfg, mesh=host.Mesh.disk(32))
    ms, kernel = _flushed_epoch_ms(hp, device)
    return {"cells": hp.E, "n_test": hp.T, "n_quad": hp.Q, "sensors": hp.n_sen, "layers": [2, 30, 30, 30, 2],
            "ms_per_epoch": ms, "kernel": kernel, "quad_pt_evals_per_s": hp.n_int / (ms * 1e-3),
            "l2": "flushed between timed epochs"}


def _c3_contraction(device, pk):
    """The split path's contraction (cells larger than a tile: C3's 10x10
    test functions on 40x40 Gauss points, 64 cells) on device-resident
    derivatives, L2 flushed per launch: contract_rowreg_kernel (warp-owned
    rows) + contract_rowreg_reduce_kernel (the per-cell sum of the CTA
    partials), against the measured HBM copy bandwidth."""
    from paper_2404_12063_b200 import gpu as G, host
    cfg = {"problem": {"forcing": "sin4pi_f", "boundary_g": "sin4pi_u", "n_boundary_points": 400},
           "discretization": {"n_test_per_dim": 10, "n_quad_per_dim": 40},
           "network": {"layers": [2, 30, 30, 30, 1]},
           "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    hp = host.HostProblem(cfg, mesh=host.Mesh.structured(8, 8))
    g = G.GpuStep.from_problem(hp.view(device), keepalive=hp)
    ms_all, ms, nbytes = g.time_contract_kernels(20)
    g.close()
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": "contract_rowreg_kernel (C3: 64 cells, T = 100, Q = 1,600)",
            "achieved": gbs, "peak": pk.get("hbm_gbs"), "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
            "traffic": (_traffic("contract_rowreg_kernel") or {}).get("bytes"),
            "bytes_per_launch": nbytes, "ms_per_launch": ms, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
            "with_partial_sum": {"kernels": "+ contract_rowreg_reduce_kernel", "ms": ms_all,
                                 "achieved": nbytes / (ms_all * 1e-3) / 1e9}}


def _sweep(device):
    """C2: unit-square cell-count sweep 1..4096 cells at T=25, Q=100."""
    from paper_2404_12063_b200 import host
    cfg = {"problem": {"forcing": "sin2pi_f", "boundary_g": "sin2pi_u", "n_boundary_points": 400},
           "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
           "network": {"layers": [2, 30, 30, 30, 1]},
           "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    out = []
    for e in (1, 2, 4, 8, 16, 32, 64):
        r = host.bench_case(cfg, e, 5, 10, 0.0, 15, device)
        out.append({"cells": e * e, "median_ms": 1e3 * r["median_s"], "p10_ms": 1e3 * r["p10_s"],
                    "p90_ms": 1e3 * r["p90_s"], "quad_pt_evals_per_s": e * e * 100 / r["median_s"]})
    return out


def _sweep_c3(device):
    """C3: high-frequency Poisson (sin4pi) p/q refinement on 8x8 cells: test
    functions 5..10 per dimension, quadrature 10..40 per dimension (Q > 128
    takes the split path: forward, standalone contraction, reverse)."""
    from paper_2404_12063_b200 import host
    cfg = {"problem": {"forcing": "sin4pi_f", "boundary_g": "sin4pi_u", "n_boundary_points": 400},
           "discretization": {"n_test_per_dim": 5, "n_quad_per_dim": 10},
           "network": {"layers": [2, 30, 30, 30, 1]},
           "training": {"learning_rate": 1e-3, "seed": 42, "precision": "single"}}
    out = []
    for t, q in ((5, 10), (8, 20), (10, 20), (10, 40)):
        r = host.bench_case(cfg, 8, t, q, 0.0, 15, device)
        out.append({"cells": 64, "n_test": t * t, "n_quad": q * q, "median_ms": 1e3 * r["median_s"],
                    "quad_pt_evals_per_s": 64 * q * q / r["median_s"]})
    return out


if __name__ == "__main__":
    main()
