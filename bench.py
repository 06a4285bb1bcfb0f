#!/usr/bin/env python
"""Benchmark: ASPOT iterations/s at BASELINE.json configs[2] (n = 16384,
fp32, squared-Euclidean cost regenerated on the fly), plus time-to-eps, the
roofline of the hot sweep kernel and the CPU oracle beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one accepted ASPOT iteration (solvers.hpp:323-369) on the
resident problem. `value` is whole-job iterations/s from CUDA-event device
time of exactly K steps (max over ranks); `e2e` is the same metric through
the public API from host buffers (upload + setup + K iterations + rounding +
download). N > 1 (torchrun, one process per GPU): the SAME problem is
row-block sharded over the N GPUs (csrc/shard.cuh: each rank sweeps n/N
rows, one NCCL all-reduce per sweep) — strong scaling of one solve; `value`
is that solve's iterations/s from the max-over-ranks device time.
"""
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

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--epsilon", type=float, default=1e-2)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work in the all-threads CPU sample")
    ap.add_argument("--ref-budget", type=float, default=90.0, help="seconds of oracle work in the --impl reference arm")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tte", action="store_true", help="skip the time-to-eps solve")
    return ap.parse_args()


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    (pynvml, every 5 ms) or, without it, nvidia-smi."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NVML_REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, [reasons])
        self._stop = threading.Event()
        self._t = None
        self.source = "nvidia-smi"
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self._nvml = pynvml
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        return float(sm), float(mx), [name for b, name in self.NVML_REASONS.items() if bits & b]

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
        if out.returncode != 0 or not out.stdout.strip():
            return None
        f = [x.strip() for x in out.stdout.strip().split(",")]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [names[k] for k in range(4) if len(f) > 4 + k and "Active" in f[4 + k] and "Not" not in f[4 + k]]
        num = lambda x: float(x) if x.replace(".", "").isdigit() else None  # noqa: E731
        return num(f[0]), num(f[1]), reasons

    def _run(self):
        while not self._stop.is_set():
            try:
                smp = self._sample_nvml() if self._nvml else self._sample_smi()
                if smp:
                    self.samples.append(smp)
            except Exception:
                pass
            self._stop.wait(0.005 if self._nvml else 0.02)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [x[0] for x in self.samples if x[0]]
        mx = [x[1] for x in self.samples if x[1]]
        reasons = sorted({r for x in self.samples for r in x[2]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples), "source": self.source}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1 and args.impl != "reference":  # the reference arm is host-only (rank 0 runs it)
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
    return rank, world, local, dist


def barrier(dist):
    if dist is not None:
        dist.barrier()


def max_over_ranks(x, dist, local):
    if dist is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def workload_points(args, product: bool):
    """The C3 instance (BASELINE configs[2]) as fp32-rounded points. The
    product arm builds it through the package; the reference arm through the
    fixture generator linked into the oracle library (same synthetic.cpp,
    identical bits), so `--impl reference` never loads libpotgpu.so."""
    import numpy as np
    if product:
        from paper_2601_17196_b200 import pot
        inst = pot.config_instance(3, n=args.n, seed=args.seed)
        if inst.cost_scale is None or inst.cost_scale <= 0:
            inst.cost_scale = pot.points_scale(inst.X, inst.Y)
        return inst
    from oracle import binding
    r, c, X, Y, s, _ = binding.config_points(3, args.n, args.seed)
    X = X.astype(np.float32).astype(np.float64)  # pot.config_instance's fp32 rounding
    Y = Y.astype(np.float32).astype(np.float64)
    m = 0.0
    for a in range(0, X.shape[0], 1024):  # pot.points_scale's association
        D = np.zeros((min(1024, X.shape[0] - a), Y.shape[0]))
        for k in range(3):
            t = X[a:a + 1024, k][:, None] - Y[:, k][None, :]
            D = D + t * t
        m = max(m, float(D.max()))
    return {"r": r, "c": c, "s": s, "X": X, "Y": Y, "cost_scale": 1.0 / m if m > 0 else 1.0, "n": args.n}


def cpu_reference(w, args, threads, budget_s=None, max_iters=None):
    """The reference solver's CPU restatement (the oracle, kind "port": the
    reference itself cannot be built here) timed on a bounded
    sample of the same workload: ASPOT iterations of the same instance. One
    iteration is timed first; the sample is then as many iterations as fit
    the time budget (at least 1, at most `max_iters`). `value` = iterations /
    loop time of that sample (the oracle's own wall_seconds, which also pays
    its initial phi/grad pass)."""
    from oracle import binding
    binding.lib().oracle_set_threads(threads)

    def run(k):
        t0 = time.perf_counter()
        res = binding.solve(0, w["r"], w["c"], w["s"], X=w["X"], Y=w["Y"], scale=w["cost_scale"],
                            epsilon=args.epsilon, max_iterations=k, skip_plan=True, log_every=10 ** 9)
        return res, time.perf_counter() - t0

    res, wall = run(1)
    k = 1
    if budget_s is not None and max_iters is not None and max_iters > 1:
        k = int(max(1, min(max_iters, budget_s // max(wall, 1e-3))))
        if k > 1:
            res, wall = run(k)
    binding.lib().oracle_set_threads(1)
    it = max(res.iterations, 1)
    return {"value": it / wall, "unit": "iterations/s", "cores": threads, "kind": "port",
            "iterations": it, "seconds": wall,
            "sample": f"{it} ASPOT iteration(s) of the same n={w['n']} instance (fp64 oracle on the fp32-rounded "
                      f"coordinates, {threads} host thread(s), incl. its initial phi/grad pass), {wall:.1f} s"}


def flush_l2(local):
    import torch
    if not hasattr(flush_l2, "buf"):
        flush_l2.buf = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")  # 256 MB > L2
    flush_l2.buf.zero_()
    torch.cuda.synchronize()


def main():
    args = parse()
    rank, world, local, dist = dist_setup(args)
    n = args.n
    threads = os.cpu_count() or 1
    config = {"workload": f"BASELINE configs[2]: registration-shaped POT n={n}, fp32, on-the-fly sq-Euclidean cost, "
                          f"eps={args.epsilon}, s=0.9, ASPOT",
              "n": n, "epsilon": args.epsilon, "solver": "aspot", "cost": "on-the-fly",
              "parallelism": f"rowshard{world}" if world > 1 else "single",
              "l2": "coordinates are L2-resident by design (on-the-fly cost); L2 flushed (256 MB write) between "
                    "timed steps"}

    if args.impl == "reference":
        # the oracle port on all host threads; rank 0 only, no GPU, no libpotgpu
        if rank != 0:
            return
        w = workload_points(args, product=False)
        ref = cpu_reference(w, args, threads, budget_s=args.ref_budget, max_iters=args.steps)
        if not args.no_cpu:  # the reference's own semantics: single-threaded (proj/README.md:132-133)
            one = cpu_reference(w, args, 1)
            ref["single_thread"] = {"value": one["value"], "unit": one["unit"], "cores": 1, "sample": one["sample"]}
        line = {"impl": "reference", "metric": "ASPOT iterations/s", "value": ref["value"], "unit": "iterations/s",
                "n_gpus": world, "steps": ref["iterations"], "warmup": 0,
                "ms_per_step": 1000.0 * ref["seconds"] / ref["iterations"],
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config, "cpu_baseline": ref,
                "note": f"--steps {args.steps} requested; the CPU sample is bounded to ~{args.ref_budget:.0f} s of "
                        f"oracle work, `steps` is what ran",
                "e2e": {"value": ref["value"], "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    from paper_2601_17196_b200 import pot
    inst = workload_points(args, product=True)
    assert inst.size() == n

    import torch
    torch.cuda.set_device(local)
    ctx = pot.Context(local)
    if world > 1:
        pot.init_distributed(ctx)  # NCCL communicator for the row shards
    cfg = pot.SolverConfig(epsilon=args.epsilon, log_every=10 ** 9, max_iterations=10 ** 7, record_rounded_cost=False,
                           materialize_plan=False)
    sess = pot.Session(pot.SolverKind.Aspot, inst, cfg, ctx=ctx)
    sess.iterate(args.warmup)
    k0, a0, s0 = sess.stats()
    per_step = []
    barrier(dist)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        done = 0
        for _ in range(args.steps):
            flush_l2(local)
            ms, it, fin = sess.iterate(1)
            per_step.append(ms)
            done += it
            if fin:
                break
    torch.cuda.synchronize()
    barrier(dist)
    k1, a1, s1 = sess.stats()
    total_ms = sum(per_step)
    total_ms = max_over_ranks(total_ms, dist, local)
    value = done / (total_ms / 1000.0) if total_ms > 0 else 0.0  # one sharded solve
    sweeps_per_it = (s1 - s0) / max(done, 1)
    # roofline of the dominant kernel (the on-the-fly sweep): MUFU ex2 bound
    ms_sweep, elems, _ = sess.time_sweep(20)
    # the other n^2 pass of an iteration: the one-sided z_check' pass fused with
    # the next z_bar (K1''), for both Greenkhorn blocks (single GPU only)
    ms_one = None
    if world == 1:
        try:
            ms_one = {"u": sess.time_one_sided(0, 10), "v": sess.time_one_sided(1, 10)}
        except pot.PotError:
            ms_one = None
    clocks = clk.summary()
    sess.close()

    # stored-cost variant of the same shape (C materialised once on the
    # device, fp32, 1 GiB) for the HBM roofline of the stored sweep
    stored = None
    try:
        st_inst = pot.Instance(r=inst.r, c=inst.c, s=inst.s, X=inst.X, Y=inst.Y, cost_scale=inst.cost_scale,
                               dtype=pot.DType.F32)
        st_inst.stored = True
        ss = pot.Session(pot.SolverKind.Aspot, st_inst, cfg, ctx=ctx)
        ss.iterate(2)
        ms_st, el_st, by_st = ss.time_sweep(10)
        ss.close()
        peaks = json.load(open(MEASURED_PEAKS)) if os.path.exists(MEASURED_PEAKS) else {}
        hbm = peaks.get("hbm_gbs", 6650.0)
        stored = {"bound": "hbm", "achieved": by_st / (ms_st * 1e-3) / 1e9, "peak": hbm, "unit": "GB/s",
                  "frac": by_st / (ms_st * 1e-3) / 1e9 / hbm, "traffic": None,
                  "kernel": "sweep_f32<SrcDenseF32>", "ms_per_launch": ms_st,
                  "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s"}
    except Exception as e:  # pragma: no cover
        stored = {"error": str(e)}

    # time-to-eps (the reference's wall_seconds: solver entry -> rounded plan)
    tte = None
    if not args.no_tte:
        full = pot.aspot_solve(inst, pot.SolverConfig(epsilon=args.epsilon, log_every=10 ** 9, record_rounded_cost=False,
                                                      materialize_plan=False), ctx=ctx)
        tte = {"seconds": full.wall_seconds, "loop_seconds": full.loop_seconds, "iterations": full.iterations,
               "status": full.status.name, "final_error": full.final_error, "tolerance": full.tolerance,
               "cost": full.cost, "feasibility_gap": full.feasibility_gap}

    # the tuned-Sinkhorn baseline on the same instance (solvers.hpp:547-589, p = 4)
    tuned = None
    if not args.no_tte:
        ts = pot.tuned_sinkhorn_solve(inst, args.epsilon, 4.0, pot.SolverConfig(log_every=10 ** 9, record_rounded_cost=False,
                                                                             materialize_plan=False), ctx=ctx)
        tuned = {"seconds": ts.wall_seconds, "loop_seconds": ts.loop_seconds, "iterations": ts.iterations,
                 "status": ts.status.name, "final_error": ts.final_error, "tolerance": ts.tolerance, "cost": ts.cost,
                 "feasibility_gap": ts.feasibility_gap, "p": 4.0}

    # e2e: the public API from host buffers, K iterations per call
    e2e_cfg = pot.SolverConfig(epsilon=args.epsilon, log_every=10 ** 9, max_iterations=args.steps,
                               record_rounded_cost=False, materialize_plan=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r2 = pot.aspot_solve(inst, e2e_cfg, ctx=ctx)
    e2e_wall = time.perf_counter() - t0
    h2d = 8 * (inst.X.size + inst.Y.size + 2 * n)
    d2h = 8 * (4 * n + 1)
    e2e_wall = max_over_ranks(e2e_wall, dist, local)
    e2e_val = r2.iterations / e2e_wall

    # DRAM bytes per launch of the same kernels from the committed ncu --set full
    # captures (profiles/run_profile.sh -> profiles/summarize_ncu.py)
    ncu_sum = {}
    for rnd in sorted(os.listdir(os.path.join(ROOT, "profiles"))) if os.path.isdir(os.path.join(ROOT, "profiles")) else []:
        f = os.path.join(ROOT, "profiles", rnd, "ncu_summary.json")
        if os.path.exists(f):
            ncu_sum = json.load(open(f))
    def traffic(name):
        v = ncu_sum.get(name)
        return None if not v else v["dram_read_bytes"] + v["dram_write_bytes"]
    if isinstance(stored, dict) and "bound" in stored:
        stored["traffic"] = traffic("sweep_stored")
        stored["traffic_source"] = "ncu --set full capture committed in profiles/ (bytes per launch)"
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    mufu_peak = 16 * nsm * sm_mhz * 1e6 / 1e9  # G ex2/s at the measured clock
    achieved = elems / (ms_sweep * 1e-3) / 1e9
    roofline = {"bound": "mufu", "achieved": achieved, "peak": mufu_peak, "unit": "Gex2/s", "frac": achieved / mufu_peak,
                "traffic": traffic("sweep_points"), "kernel": "sweep_pts2_f32 (points, 2 rows x 16 columns per warp step)", "ms_per_launch": ms_sweep,
                "per_unit": "1 MUFU.EX2 per plan entry; n^2 entries per launch",
                "peak_source": f"16 ex2/clk/SM x {nsm} SMs x median SM clock {sm_mhz} MHz under load"}
    one_sided = None
    if ms_one:
        one_sided = {"bound": "mufu", "peak": mufu_peak, "unit": "Gex2/s", "traffic": traffic("sweep_pts1"),
                     "kernel": "sweep_pts1_f32 (one-sided z_check' pass fused with the next z_bar, K1'')",
                     "per_unit": "1 MUFU.EX2 per plan entry; n^2 entries per launch",
                     "ms_per_launch": ms_one,
                     "achieved": {b: elems / (ms * 1e-3) / 1e9 for b, ms in ms_one.items()},
                     "frac": {b: elems / (ms * 1e-3) / 1e9 / mufu_peak for b, ms in ms_one.items()}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        w = workload_points(args, product=False)
        cpu = cpu_reference(w, args, threads, budget_s=args.cpu_budget, max_iters=args.steps)
    if rank == 0:
        line = {"metric": "ASPOT iterations/s", "value": value, "unit": "iterations/s", "n_gpus": world,
                "steps": len(per_step), "warmup": args.warmup, "ms_per_step": total_ms / max(len(per_step), 1),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config, "clocks": clocks,
                "e2e": {"value": e2e_val, "unit": "iterations/s", "h2d_bytes_per_step": h2d / max(r2.iterations, 1),
                        "d2h_bytes_per_step": d2h / max(r2.iterations, 1),
                        "note": "one public-API call (aspot_solve, max_iterations=K) from host buffers: upload, setup, "
                                "K iterations, rounding, download"},
                "gpu_launches": k1 - k0, "sweeps_per_iteration": sweeps_per_it,
                "roofline": roofline, "roofline_one_sided": one_sided, "roofline_stored": stored, "time_to_eps": tte, "tuned_sinkhorn_time_to_eps": tuned,
                "cpu_baseline": cpu}
        print(json.dumps(line))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
