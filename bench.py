#!/usr/bin/env python
"""Benchmark of the batched A-MMMSE engine (driver contract, one JSON line).

A step = one batched solve, to convergence, of the whole workload with its
inputs resident in HBM.  Default workload: BASELINE.json configs[1]
("medium": M=64, K=16, N=2, d=2, 4096 realizations at each SNR in
{0,10,20,30} dB, i.e. 16384 realizations per step and per GPU).  Multi-GPU:
one process per GPU under torchrun, each rank solves its own 16384
realizations (global seeds rank*4096 + i per SNR block): weak scaling, no
collective on the data path; the per-realization WSR / iteration counts are
gathered to rank 0 with one NCCL all_gather at the end of each step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config medium|small|...]
    python bench.py --impl reference ...   # CPU reference arm (oracle port, host cores)
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2510_20507_b200.inputs import MEDIUM, WORKLOADS, Batch  # noqa: E402

METRIC = "channel realizations solved/sec to convergence"
UNIT = "realizations/s"


# --------------------------------------------------------------------------- workloads
def bench_workload(name: str):
    """(list of Workload blocks, label).  'medium' = the four SNR blocks."""
    if name == "medium":
        return [WORKLOADS[n] for n in MEDIUM], "medium"
    return [WORKLOADS[name]], name


def build_inputs(blocks, per_block: int, seed0: int, workers: int = 0) -> Batch:
    workers = workers or min(32, os.cpu_count() or 1)
    return Batch.concat([w.batch(B=per_block, seed0=seed0, workers=workers) for w in blocks])


def flops_per_unit(w) -> float:
    """Algorithmic work of one realization-iteration: two complex GEMMs
    G = H V and grad = H^H Yhat, F = 16 K^2 N d M real flops."""
    return 16.0 * w.K * w.K * w.N * w.d * w.M


def bytes_per_realization(w, itemsize: int) -> dict:
    c = 2 * itemsize
    h2d = w.K * w.N * w.M * c + w.K * w.M * w.d * c + 8 * (2 + w.K)
    d2h = w.K * w.M * w.d * c + 8 + 4 + 1 + 8 + 4 + 4 + 8
    return dict(h2d=h2d, d2h=d2h)


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=1)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# --------------------------------------------------------------------------- CPU arms
def cpu_sample_indices(B_block: int, n_blocks: int, n: int):
    """Round-robin over the SNR blocks so the sample mixes their iteration counts."""
    idx = []
    i = 0
    while len(idx) < n:
        for b in range(n_blocks):
            if len(idx) < n:
                idx.append(b * B_block + i)
        i += 1
    return idx


def cpu_time(blocks, batch: Batch, per_block: int, target_s: float, pool):
    """Rounds of `workers` realizations (one per process) until >= target_s of
    wall time; returns realizations / second over all rounds."""
    from oracle.cpu_baseline import tasks_from_batch, time_tasks

    w = blocks[0]
    opts = dict(eps1=w.eps1, eps2=w.eps2, max_iters=w.max_iters)
    order = cpu_sample_indices(per_block, len(blocks), batch.B)
    n = t = iters = 0
    while t < target_s and n < batch.B:
        idx = order[n:n + pool.workers]
        dt, out = time_tasks(pool, tasks_from_batch(batch, idx, opts))
        n += len(idx)
        t += dt
        iters += sum(o[1] for o in out)
    return dict(value=n / t, seconds=t, n=n, iters=iters)


def run_reference_arm(args, rank: int):
    """--impl reference: the oracle port (reference algorithm, complex128
    numpy/scipy) on the host cores, same workload / metric / unit."""
    if rank != 0:
        return
    from oracle.cpu_baseline import CpuPool

    blocks, label = bench_workload(args.config)
    per_block = min(blocks[0].B, 512)
    batch = build_inputs(blocks, per_block, 0)
    pool = CpuPool()
    step_s = args.cpu_seconds
    for _ in range(args.warmup):
        cpu_time(blocks, batch, per_block, min(step_s, 5.0), pool)
    vals, secs, ns = [], [], []
    for _ in range(args.steps):
        r = cpu_time(blocks, batch, per_block, step_s, pool)
        vals.append(r["value"])
        secs.append(r["seconds"])
        ns.append(r["n"])
    pool.close()
    value = float(np.mean(vals))
    w = blocks[0]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded Philox, SURVEY.md §8(d))",
        "config": {"workload": label, "M": w.M, "K": w.K, "N": w.N, "d": w.d,
                   "realizations_per_step": int(np.mean(ns)), "max_iters": w.max_iters,
                   "eps2": w.eps2, "gamma": [b.gamma for b in blocks], "omega": w.omega},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                         "sample": f"{int(np.mean(ns))} realizations per step (round-robin over "
                                   f"the SNR blocks), oracle/ammmse_oracle.py in a "
                                   f"{os.cpu_count()}-process pool, 1 BLAS thread each"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="medium")
    ap.add_argument("--per-block", type=int, default=None, help="realizations per SNR block")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--device-inputs", action="store_true",
                    help="generate the (i.i.d.) workload on the device at its full batch size")
    ap.add_argument("--e2e-chunks", type=int, default=8,
                    help="slices of the pipelined host-buffer solve in the e2e measurement")
    ap.add_argument("--no-phase-profile", action="store_true",
                    help="skip the extra instrumented launch (bcgd_step share)")
    ap.add_argument("--cluster-size", type=int, default=0, help="engine knob (0 = automatic)")
    ap.add_argument("--h-placement", type=int, default=0, help="engine knob (0 = automatic)")
    ap.add_argument("--tensor-cores", type=int, default=0, help="engine knob (0 auto, 1 on, 2 off)")
    ap.add_argument("--gen-workers", type=int, default=0,
                    help="processes for host input generation (1 under ncu)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2510_20507_b200.solvers import AmmmseEngine

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    blocks, label = bench_workload(args.config)
    w = blocks[0]
    per_block = args.per_block or w.B
    eng = AmmmseEngine(dev)
    to = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    itemsize = np.dtype(w.dtype).itemsize // 2
    if args.device_inputs:
        # the workload at its full BASELINE batch, generated on the device
        # (ammmse_generate_iid / generate_kronecker; distributionally, not bit-,
        # identical to the host generators); the CPU baseline still runs on a
        # host-generated sample
        gen = lambda b: (eng.generate_iid if b.channel == "iid" else eng.generate_kronecker)
        parts = [gen(b)(per_block, b.K, b.N, b.M, b.d, seed0=rank * per_block, p_max=b.p_max,
                        weights=b.weights, dtype=np.dtype(b.dtype).name) for b in blocks]
        dH = torch.cat([p[0] for p in parts])
        dV0 = torch.cat([p[1] for p in parts])
        dA = torch.cat([p[2] for p in parts])
        B = dH.shape[0]
        ds2 = torch.ones(B, dtype=torch.float64, device=dev)
        dP = torch.cat([torch.full((per_block,), b.p_max, dtype=torch.float64, device=dev)
                        for b in blocks])
        g_arr = torch.cat([torch.full((per_block,), b.gamma, dtype=torch.float64, device=dev)
                           for b in blocks])
        o_arr = torch.cat([torch.full((per_block,), b.omega, dtype=torch.float64, device=dev)
                           for b in blocks])
        del parts
        cpu_pb = min(per_block, 256)
        batch = build_inputs(blocks, cpu_pb, seed0=0, workers=args.gen_workers)
        args.no_e2e = True  # inputs are created on the device: no host-buffer e2e number
    else:
        cpu_pb = per_block
        batch = build_inputs(blocks, per_block, seed0=rank * per_block, workers=args.gen_workers)
        B = batch.B
        dH, ds2, dP, dA, dV0 = (to(batch.channels), to(batch.noise_power), to(batch.p_max),
                                to(batch.weights), to(batch.init_precoders))
        g_arr, o_arr = to(batch.gamma), to(batch.omega)
    # per-realization (gamma, omega): each SNR block carries its own step
    kw = dict(gamma=g_arr, omega=o_arr, eps1=w.eps1, eps2=w.eps2,
              max_iters=w.max_iters, cluster_size=args.cluster_size, h_placement=args.h_placement,
              tensor_cores=args.tensor_cores)
    stream = torch.cuda.current_stream(dev)

    gather_buf = torch.empty((world, B, 2), dtype=torch.float64, device=dev) if world > 1 else None

    def step(out=None):
        res = eng.solve(dH, ds2, dP, dA, dV0, out=out, stream=stream, **kw)
        if world > 1:  # final gather of per-realization WSR / iterations (the only collective)
            local_res = torch.stack([res.wsr_bits, res.iterations.to(torch.float64)], dim=1)
            dist.all_gather_into_tensor(gather_buf.view(world * B, 2), local_res)
        return res

    res = None
    for _ in range(max(args.warmup, 0)):
        res = step(res)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res = step(res)
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * B / (ms_per_step * 1e-3)

    host = res.to_host()
    iters_total = int(host.iterations.sum())
    n_bad = int((host.status != 0).sum())

    # ---- end to end through the public API with host buffers (pinned) ----
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        hH, hs2, hP, hA, hV0 = (pin(batch.channels), pin(batch.noise_power), pin(batch.p_max),
                                pin(batch.weights), pin(batch.init_precoders))
        hout = {k: torch.empty(tuple(getattr(res, k).shape), dtype=getattr(res, k).dtype).pin_memory()
                for k in ("final_precoders", "wsr_bits", "iterations", "converged",
                          "stationarity_residual", "switch_iteration", "status")}
        dbufs = [torch.empty_like(x, device=dev) for x in (hH, hs2, hP, hA, hV0)]

        # slices of at least 2048 realizations (a tiny batch is one launch)
        e2e_chunks = max(1, min(args.e2e_chunks, B // 2048))

        def e2e_step():
            # public API, host buffers: H2D of slice i+1 and D2H of slice i-1
            # overlap the solve of slice i (AmmmseEngine.solve_host)
            r = eng.solve_host((hH, hs2, hP, hA, hV0), hout, dbufs, res, stream=stream,
                               chunks=e2e_chunks, **kw)
            if world > 1:
                local_res = torch.stack([r.wsr_bits, r.iterations.to(torch.float64)], dim=1)
                dist.all_gather_into_tensor(gather_buf.view(world * B, 2), local_res)
            return r

        for _ in range(2):
            e2e_step()
        barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
        barrier()
        ems = f0.elapsed_time(f1)
        if world > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        h2d = sum(x.numel() * x.element_size() for x in (hH, hs2, hP, hA, hV0))
        d2h = sum(x.numel() * x.element_size() for x in hout.values())
        e2e = {"value": world * B / (ems / args.steps * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if rank != 0:
        if world > 1:
            dist.barrier(device_ids=[local])
            dist.destroy_process_group()
        return

    # ---- roofline of the (only) kernel: FMA pipe, GEMM-step flops ----
    import ctypes

    probe = ctypes.CDLL(os.path.join(ROOT, "paper_2510_20507_b200", "libammmse_probe.so"))
    probe.ammmse_probe_fp32_flops.restype = ctypes.c_double
    probe.ammmse_probe_fp64_flops.restype = ctypes.c_double
    peak32 = probe.ammmse_probe_fp32_flops(400)
    peak64 = probe.ammmse_probe_fp64_flops(100)
    fpu = flops_per_unit(w)
    achieved = fpu * iters_total / (ms_per_step * 1e-3)  # rank 0's launch, rank 0's units
    if world > 1:
        achieved = fpu * iters_total / (ms_per_step * 1e-3)
    peak = peak32 if w.dtype == np.complex64 else peak64
    roofline = {
        "bound": "fma", "pipe": "fp32 FFMA (CUDA cores)" if w.dtype == np.complex64 else "fp64 DFMA",
        "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
        "frac": achieved / peak if peak > 0 else None, "traffic": None,
        "peak_source": "measured live by libammmse_probe (register FFMA/DFMA throughput kernel)",
        "work": f"F=16*K^2*N*d*M={fpu:.0f} flop per realization-iteration x {iters_total} "
                f"realization-iterations per launch",
        "kernel": "ammmse_solve_kernel (1 launch per step)",
    }

    # BCGD-step share of the kernel (GEMM-step fraction =
    # F x realization-iterations / t_GEMM / peak): one extra, untimed solve with
    # the engine's phase timers (thread-0 clock64 per phase), after the timed region.
    if not args.no_phase_profile:
        import ctypes

        from paper_2510_20507_b200 import _native

        os.environ["AMMMSE_PROFILE_PHASES"] = "1"
        eng.solve(dH, ds2, dP, dA, dV0, out=res, stream=stream, **kw)
        torch.cuda.synchronize()
        del os.environ["AMMMSE_PROFILE_PHASES"]
        sh = (ctypes.c_double * 16)()
        f0, nb = ctypes.c_int(), ctypes.c_int()
        n = _native.lib().ammmse_last_phase_profile(sh, 16, ctypes.byref(f0), ctypes.byref(nb))
        if n > 0:
            share = sum(sh[f0.value + i] for i in range(nb.value))
            roofline["bcgd_step"] = {
                "share_of_kernel": share, "frac": roofline["frac"] / share if share > 0 else None,
                "achieved": roofline["achieved"] / share if share > 0 else None,
                "phases": [round(sh[i], 4) for i in range(n)],
                "note": "F x realization-iterations / time in the BCGD step phases (GEMM-A + "
                        "step + projection, GEMM-B) / peak; phase shares from thread-0 clock64 "
                        "timers of one extra untimed launch"}

    # DRAM traffic of the same kernel from the committed ncu --set full capture
    # (profiles/ncu_traffic.json, per realization), scaled to this launch, next
    # to the algorithmic bytes (H and V0 read once, V_out written once).
    tdb_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tdb = json.load(open(tdb_path)) if os.path.exists(tdb_path) else {}
    bpr = bytes_per_realization(w, itemsize)
    roofline["algorithmic_bytes"] = int(B * (bpr["h2d"] + bpr["d2h"]))
    if label in tdb:
        ent = tdb[label]
        roofline["traffic"] = int(ent["bytes_per_realization"] * B)
        roofline["traffic_source"] = (f"{ent['source']}: ncu dram__bytes_read+write of "
                                      f"{ent['realizations']} realizations, scaled to {B}")

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        from oracle.cpu_baseline import CpuPool

        pool = CpuPool()
        r = cpu_time(blocks, batch, cpu_pb, args.cpu_seconds, pool)
        pool.close()
        cpu = {"value": r["value"], "unit": UNIT, "cores": pool.workers, "kind": "port",
               "sample": f"{r['n']} realizations (round-robin over the SNR blocks, "
                         f"{r['iters']} realization-iterations, {r['seconds']:.1f} s) of this "
                         f"workload, oracle/ammmse_oracle.py (complex128) in a "
                         f"{pool.workers}-process pool, 1 BLAS thread each"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "c64 (fp32 GEMM, fp64 Gram/log-det/WSR)" if w.dtype == np.complex64 else "c128",
        "data": ("synthetic, generated on the device (Philox4x32-10 CN(0,1), ammmse_generate_iid)"
                 if args.device_inputs else "synthetic (seeded Philox inputs, SURVEY.md §8(d))"),
        "config": {"workload": label, "M": w.M, "K": w.K, "N": w.N, "d": w.d,
                   "realizations_per_gpu_step": B, "snr_blocks": len(blocks),
                   "max_iters": w.max_iters, "eps2": w.eps2, "gamma": [b.gamma for b in blocks],
                   "omega": w.omega,
                   "mean_iterations": iters_total / B, "failed_realizations": n_bad,
                   "parallelism": f"dp{world} (realizations sharded, no data-path collective)",
                   "l2": f"inputs larger than L2: {dH.numel() * dH.element_size() / 2**20:.0f} MiB "
                         f"of channels read once per step"},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
