"""Benchmark of the DQN learner update (BASELINE.json metric: learner
updates/s and sampled transitions/s, Dueling+Double+PER, batch 32, 1M
synthetic Atari transitions).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode auto|single|dp|replicas]

Our arm (default) prints ONE JSON line on rank 0:
  value      device-timed updates/s, inputs (ring, tree, pre-drawn uniforms)
             resident in HBM, each step one CUDA-graph replay of the whole
             update (+ amortised target sync every 2,500 updates);
  e2e        the same metric through the public API ``learn_step(online,
             target, memory, optimizer, config, step, rng)``: host draws ->
             pinned H2D -> graph -> D2H TdResult -> numpy, every step;
  roofline   the dominant layer phase (GEMM) of the step, timed alone with
             CUDA events on its stream, vs MEASURED_PEAKS.json;
  cpu_baseline  the CPU oracle port of the reference learn_step on this
             host's cores for a bounded sample (all BLAS threads, and one
             pinned core under ``single_core``).
``--impl reference`` times that CPU path alone and prints its own line; it
never imports this package (the synthetic data generator is loaded from its
file), so no CUDA library of ours is loaded in that arm.

Multi-GPU.  ``--gpus N`` (N > 1) outside torchrun launches N ranks itself
through torch.distributed.run (and refuses when fewer than N GPUs are
visible); under torchrun each rank reads RANK / WORLD_SIZE / LOCAL_RANK.  The
default for N > 1 is the cfg5 data-parallel learner (``--mode dp``,
paper_1804_05834_b200/dp.py: replay sharded across the ranks, global
stratified PER over all-gathered shard totals, per-GPU batch 32, frames read
from the owners' rings over NVLink, NCCL gradient all-reduce, one CUDA graph
per rank and update); ``--mode replicas`` runs N independent learners (the
population of seeds, no data-path collective).  Both are weak scaling; rank 0
reports the max-over-ranks device time.  NCCL_DEBUG=INFO (INIT, ENV) goes to
stderr for N > 1.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "learner_updates_per_sec"
UNIT = "updates/s"
T_ROOF_US = 7.48     # 49.06 MB / 6562.6 GB/s per cfg4 update

CONFIGS = {
    "cfg1": dict(dueling=False, double=False, per=False, capacity=10_000,
                 desc="Nature DQN, uniform replay 10k, batch 32"),
    "cfg2": dict(dueling=False, double=True, per=False, capacity=1_000_000,
                 desc="Double DQN, uniform replay 1M, batch 32"),
    "cfg3": dict(dueling=False, double=True, per=True, capacity=1_000_000,
                 desc="Double DQN + PER (alpha 0.6, beta annealed), 1M, batch 32"),
    "cfg4": dict(dueling=True, double=True, per=True, capacity=1_000_000,
                 desc="Dueling + Double + PER, 1M transitions, batch 32, target sync 10k env steps"),
}
TARGET_SYNC_UPDATES = 10_000 // 4      # target_sync env steps / update_period


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def load_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu_index: int):
        self.samples, self.proc, self.gpu = [], None, gpu_index

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.samples if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        # the median under load: samples with the GPU busy (an idle GPU drops its
        # clocks; host-side setup inside a sampled region would otherwise pull the
        # median down)
        busy = [r for r in rows if len(r) >= 7 and r[6].replace(".", "").isdigit()
                and float(r[6]) > 0]
        use = busy or rows
        sm = sorted(float(r[0]) for r in use)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in use for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(use), "idle_samples": len(rows) - len(busy) if busy else 0}


# --------------------------------------------------------------------------
# CPU side: the oracle port of the reference learn_step
# --------------------------------------------------------------------------

def load_synth():
    """The synthetic-data generator, loaded straight from its file so the CPU
    arm never imports the package (whose __init__ loads libdqn_b200.so)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "dqn_bench_synth", REPO / "paper_1804_05834_b200" / "synth.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def cpu_learner(cfg_name: str, batch: int = 32, seed: int = 0, pool: int = 2048):
    """Oracle learner at the bench config.  The 1M-leaf fp64 tree is real; the
    frame store is a pool of ``pool`` synthetic transitions addressed by
    slot % pool (the reference's float32 ring would need 226 GB of host RAM;
    gather cost per sample is unchanged: one fancy-index copy per state)."""
    from oracle import deepq_oracle as O
    synth = load_synth()
    c = CONFIGS[cfg_name]
    cap = c["capacity"]
    shape = (84, 84, 4)

    class PooledRing(O.Ring):
        def __init__(self):
            self.capacity, self.state_shape = cap, shape
            sl = np.arange(pool)
            self.states = synth.frames(seed, 0, sl)
            self.next_states = synth.frames(seed, 1, sl)
            a, r, t = synth.metadata(seed, cap)
            self.actions, self.rewards, self.terminals = a, r, t
            self.cursor, self.size = 0, cap

        def gather(self, idx, prob, w):
            p = idx % pool
            return O.Batch(self.lift(self.states[p]), self.actions[idx], self.rewards[idx].copy(),
                           self.lift(self.next_states[p]), self.terminals[idx], idx, prob, w)

    on = O.QNet(O.ATARI_TRUNK, shape, 4, c["dueling"])
    tg = O.QNet(O.ATARI_TRUNK, shape, 4, c["dueling"])
    on.init(np.random.SeedSequence([seed, 3]))
    tg.copy_from(on)
    opt = O.RmsPropState(on)
    ring = PooledRing()
    if c["per"]:
        mem = O.PerReplay(cap, shape, 0.6, 0.01, (0.4, 1.0, 50_000_000))
        mem.ring = ring
        td = synth.warmup_td(seed, cap)
        mem.tree.nodes[mem.tree.base:mem.tree.base + cap] = (td + 0.01) ** 0.6
        mem.tree.rebuild()
        mem.max_priority = float((td + 0.01).max())
    else:
        mem = ring
    lcfg = O.LearnCfg(double=c["double"], batch_size=batch)
    return on, tg, mem, opt, lcfg, O


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 1) for d in threadpool_info() if d.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_time(cfg_name: str, steps: int, warmup: int, budget_s: float | None, batch: int = 32):
    """Time the oracle learn_step; returns (updates/s, steps timed)."""
    on, tg, mem, opt, lcfg, O = cpu_learner(cfg_name, batch)
    rng = np.random.default_rng(np.random.SeedSequence([0, 2]))
    for s in range(warmup):
        O.learn_step(on, tg, mem, opt, lcfg, 50_000 + s, rng=rng)
    t0 = time.perf_counter()
    n = 0
    while True:
        O.learn_step(on, tg, mem, opt, lcfg, 50_000 + warmup + n, rng=rng)
        n += 1
        el = time.perf_counter() - t0
        if budget_s is None and n >= steps:
            break
        if budget_s is not None and (el >= budget_s or n >= steps):
            break
    return n / (time.perf_counter() - t0), n


def cpu_time_single_core(cfg_name: str, steps: int, warmup: int, budget_s: float | None,
                         batch: int = 32):
    """The same, pinned to one core with one BLAS thread (BASELINE.md §3.1's
    1-core setting: taskset -c <cpu> + OPENBLAS_NUM_THREADS=1)."""
    from threadpoolctl import threadpool_limits
    cpus = sorted(os.sched_getaffinity(0))
    try:
        os.sched_setaffinity(0, {cpus[0]})
        with threadpool_limits(limits=1):
            return cpu_time(cfg_name, steps, warmup, budget_s, batch)
    finally:
        os.sched_setaffinity(0, set(cpus))


def cpu_baseline_obj(cfg_name: str, batch: int, steps: int, warmup: int,
                     budget_s: float | None, budget_1core_s: float | None) -> dict:
    """cpu_baseline: the oracle port of the reference learn_step on this host,
    all BLAS threads (value) and one pinned core (single_core)."""
    ups, n = cpu_time(cfg_name, steps, warmup, budget_s, batch)
    cores = blas_threads()
    ups1, n1 = cpu_time_single_core(cfg_name, max(3, steps // 3), 2, budget_1core_s, batch)
    what = (f"({cfg_name}, batch {batch}, 1M-leaf fp64 tree, pooled frame store, "
            f"numpy/OpenBLAS")
    return {"value": ups, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{n} oracle learn_step updates {what} {cores} threads)",
            "cpu": cpu_model(), "nproc": os.cpu_count(),
            "single_core": {"value": ups1, "unit": UNIT, "cores": 1,
                            "sample": f"{n1} oracle learn_step updates {what} 1 thread, "
                                      f"pinned to one core)"}}


def bench_config(cfg_name: str, capacity: int, batch: int, world: int, mode: str) -> dict:
    """The ``config`` object, identical in both arms for the same command."""
    c = CONFIGS[cfg_name]
    if world == 1 and mode != "dp":
        workload, par = c["desc"], "single GPU"
    elif mode == "replicas":
        workload, par = c["desc"] + f" (population of {world} independent learners)", \
            f"replicas x{world}"
    else:
        workload = (f"cfg5: Dueling + Double + PER data-parallel, replay sharded over {world} "
                    f"GPUs, per-GPU batch {batch}")
        par = f"dp{world}"
    return {"workload": workload, "capacity": capacity, "global_batch": batch * world,
            "per_gpu_batch": batch, "parallelism": par,
            "l2": "inputs larger than L2 (56 GB u8 ring); parameters stay L2-resident across "
                  "updates as in training"}


def run_reference(args):
    """--impl reference: the reference learn_step's CPU path (the oracle port,
    see module doc) on this host, on the same config / metric / unit as our
    arm.  At N > 1 the comparator is cfg5's global batch 32 N in one process
    (the reference has no data-parallel mode), its value counted in the same
    unit as our DP arm (batch-32 learner updates/s = global updates/s x N)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    n_gpus = max(world, args.gpus)
    mode = resolve_mode(args, n_gpus)
    per_rank = n_gpus if mode == "dp" else 1
    batch = args.batch * per_rank
    cap = args.capacity or CONFIGS[args.config]["capacity"]
    ups, n = cpu_time(args.config, args.steps, args.warmup, None, batch)
    cores = blas_threads()
    ups1, n1 = cpu_time_single_core(args.config, max(3, args.steps // 4), 2, 20.0, batch)
    value = ups * per_rank if mode == "dp" else ups
    what = (f"({args.config}, batch {batch}, 1M-leaf fp64 tree, pooled frame store) after "
            f"{args.warmup} warm-up, numpy/OpenBLAS")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus,
        "steps": n, "warmup": args.warmup, "ms_per_step": 1000.0 / ups, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args.config, cap, args.batch, n_gpus, mode),
        "transitions_per_sec": ups * batch,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n} oracle learn_step updates {what} {cores} threads",
                         "cpu": cpu_model(), "nproc": os.cpu_count(),
                         "single_core": {"value": ups1 * (per_rank if mode == "dp" else 1),
                                         "unit": UNIT, "cores": 1,
                                         "sample": f"{n1} updates {what} 1 thread, pinned"}},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if mode == "dp":
        line["note"] = (f"the reference has no data-parallel mode: one learn_step at global batch "
                        f"{batch} per step, value = updates/s x {per_rank} (batch-{args.batch} "
                        f"learner updates/s, our DP arm's unit)")
    elif mode == "replicas":
        line["note"] = "one CPU learner; the population mode's value on the GPU arm is summed over GPUs"
    print(json.dumps(line), flush=True)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# --------------------------------------------------------------------------
# GPU side
# --------------------------------------------------------------------------

def gemm_flops(u: dict, batch: int, phase: int) -> float:
    """Algorithmic FLOPs (2 per MAC) of one layer phase at ``batch``."""
    os_ = u["out_shape"]
    oh, ow, n = os_ if len(os_) == 3 else (1, 1, os_[0])
    if u["kind"] == 2:                       # dueling head: value + advantages
        n += 1
    h, w, c = u["in_shape"]
    fh, fw, sh, sw = u["geo"]
    if phase == 1 and (sh > 1 or sw > 1):
        # strided dgrad: an input pixel receives (fh/sh)*(fw/sw) taps (interior)
        return 2.0 * batch * h * w * c * n * (fh // sh) * (fw // sw)
    return 2.0 * batch * oh * ow * n * fh * fw * c


def layer_roofline(P, on, plan, peaks, peak_kind, reps=50):
    """Time every layer phase of the online net at its learner batch alone
    (CUDA events on the launching stream) and report the dominant one."""
    import ctypes as C
    import torch
    from paper_1804_05834_b200 import _lib
    st = torch.cuda.current_stream()
    best = None
    rows = []
    for li, u in enumerate(on._units):
        for phase in (0, 1, 2):
            if phase == 1 and li == 0:
                continue                         # the learner skips conv1 dX
            bind = plan.on_bind if phase == 0 else plan.on_view
            batch = bind.batch
            desc = on.desc_for(bind.x)
            args = (_lib.stream_ptr(), C.byref(desc), on.flat_values.data_ptr(),
                    on.flat_grads.data_ptr(), C.byref(bind.struct), li, phase,
                    plan.flags.data_ptr())
            for _ in range(3):
                _lib.call("dqn_net_layer", *args)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(reps):
                _lib.call("dqn_net_layer", *args)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            fl = gemm_flops(u, batch, phase)
            rows.append({"layer": u["name"], "phase": ["fwd", "dgrad", "wgrad"][phase],
                         "batch": batch, "us": ms * 1e3, "gflop": fl / 1e9})
            if best is None or ms > best[0]:
                best = (ms, u["name"], phase, fl, batch)
    on.flat_grads.zero_()
    ms, name, phase, fl, batch = best
    achieved = fl / (ms * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"])
    label = f"{name}.{['fwd', 'dgrad', 'wgrad'][phase]} (batch {batch})"
    traffic, traffic_src = None, None
    try:      # dram__bytes_read + dram__bytes_write per launch from a committed ncu capture
        t = json.load(open(REPO / "profiles" / "roofline_traffic.json"))
        if label in t.get("kernels", {}):
            traffic, traffic_src = t["kernels"][label]["dram_bytes"], t.get("source")
    except (OSError, ValueError):
        pass
    return {"kernel": label,
            "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": f"{peak_kind} bf16 dense burst",
            "algorithmic_flop_per_launch": fl, "avg_launch_us": ms * 1e3}, rows


def run_ours(args):
    import torch
    import paper_1804_05834_b200 as P
    from paper_1804_05834_b200 import _lib, agent

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    c = CONFIGS[args.config]
    cap = args.capacity or c["capacity"]
    k = args.batch
    seed = 1 + rank
    cfg = P.RunConfig(batch_size=k, double=c["double"], dueling=c["dueling"],
                      priority_alpha=0.6 if c["per"] else 0.0, beta_end_step=50_000_000)
    on = P.build_network("atari", (84, 84, 4), 4, c["dueling"])
    tg = P.build_network("atari", (84, 84, 4), 4, c["dueling"])
    P.init_params(on, np.random.SeedSequence([seed, 3]))
    P.sync_target(on, tg)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    t_fill = time.perf_counter()
    if c["per"]:
        mem = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()))
    else:
        mem = P.ReplayMemory(cap, (84, 84, 4))
    mem.fill_synthetic(seed, cap)
    torch.cuda.synchronize()
    t_fill = time.perf_counter() - t_fill

    rng = np.random.default_rng(np.random.SeedSequence([seed, 2]))
    step0 = 50_000
    # --- warm-up through the public API (first call eager, then capture) ---
    for s in range(max(args.warmup, 3)):
        P.learn_step(on, tg, mem, opt, cfg, step0 + s, rng)
    plan = agent._plan_for(on, tg, mem, opt, cfg)
    assert plan.graph is not None, "learn_step graph was not captured"

    # launches per update (count one eager enqueue)
    n0 = _lib.lib.dqn_launch_count()
    agent.USE_GRAPH = False
    P.learn_step(on, tg, mem, opt, cfg, step0 + 100, rng)
    agent.USE_GRAPH = True
    launches_per_step = int(_lib.lib.dqn_launch_count() - n0)

    # --- device-resident loop: pre-drawn inputs in HBM, one graph per step ---
    K = args.steps
    if plan.per:
        draws = np.empty((K, k + 1))
        for s in range(K):
            draws[s, :k] = rng.random(k)
            draws[s, k] = mem.beta(step0 + 200 + s)
    else:
        draws = np.stack([rng.integers(0, mem.size, size=k) for _ in range(K)]).astype(np.int64)
    d_draws = torch.as_tensor(draws, device="cuda")
    # a copy of the graph without the host copies: capture enqueue() with
    # device-side inputs
    saved_in = (plan.h_in, plan.h_idx)
    slot = torch.zeros_like(d_draws[0])
    if plan.per:
        plan.h_in = slot
    else:
        plan.h_idx = slot
    # same capture stream / node priorities as learn_step's own graph
    g_keep, g = agent.capture_graph(lambda: plan.enqueue(io=False), plan.capture_stream)
    plan.h_in, plan.h_idx = saved_in
    sp = torch.cuda.current_stream().cuda_stream
    stream = torch.cuda.current_stream()
    peaks, peak_kind = load_peaks()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for s in range(K):
            slot.copy_(d_draws[s], non_blocking=True)
            g.launch(sp)
            if (s + 1) % TARGET_SYNC_UPDATES == 0:
                P.sync_target(on, tg)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / K
    value = world * K / (ms / 1e3)

    # --- e2e through the public API with host draws and host results ---
    torch.cuda.synchronize()
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    t0 = time.perf_counter()
    for s in range(K):
        res = P.learn_step(on, tg, mem, opt, cfg, step0 + 300 + s, rng)
        if (s + 1) % TARGET_SYNC_UPDATES == 0:
            P.sync_target(on, tg)
    e3.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    ms_e2e = max(e2.elapsed_time(e3), wall * 1e3)
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e_value = world * K / (ms_e2e / 1e3)
    assert np.all(np.isfinite(res.td_errors))

    roof, rows = layer_roofline(P, on, plan, peaks, peak_kind)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_obj(args.config, k, 1 << 30, 2, args.cpu_budget, args.cpu_budget_1core)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hash-generated u8 84x84x4 frames, seeded metadata, random-init nets)",
            "config": bench_config(args.config, cap, k, world, "single" if world == 1 else "replicas"),
            "fill_seconds": round(t_fill, 2),
            "transitions_per_sec": value * k,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": plan.h2d_bytes,
                    "d2h_bytes_per_step": plan.d2h_bytes,
                    "path": "paper_1804_05834_b200.learn_step (host rng draws in pinned memory, "
                            "read by the graph's first kernel -> CUDA graph -> TdResult and flag "
                            "word written to pinned memory by the head / optimizer kernels; the "
                            "bytes crossing the host link are counted as h2d / d2h)"},
            "roofline": roof,
            "step_roofline": {"bound": "hbm", "t_roof_us": T_ROOF_US,
                              "frac": T_ROOF_US / (ms_per_step * 1e3),
                              "note": "SURVEY.md §8(d): 49.06 MB algorithmic bytes per update"},
            "layer_phases": rows,
            "gpu_launches": launches_per_step * K,
            "launches_per_step": launches_per_step,
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_dp(args):
    """cfg5: the data-parallel learner (dp.DeviceDataParallelLearner): replay
    sharded over the ranks (capacity / N each, CUDA-IPC shareable), global
    stratified PER over the shard totals, per-rank batch 32 (global 32 N),
    frames read from the owners' rings over NVLink, NCCL gradient all-reduce,
    the whole global update one CUDA graph per rank.  value = batch-32
    learner updates/s summed over the GPUs (= global updates/s x N =
    transitions/s / 32), device-timed over graph launches with the uniforms
    pre-drawn in HBM; e2e = DeviceDataParallelLearner.step with host draws
    and host results every step."""
    import torch
    import torch.distributed as dist
    import paper_1804_05834_b200 as P
    from paper_1804_05834_b200 import _lib, agent, dp

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        if "MASTER_ADDR" not in os.environ:             # plain `python bench.py --mode dp`
            import socket
            with socket.socket() as so:
                so.bind(("127.0.0.1", 0))
                os.environ["MASTER_PORT"] = str(so.getsockname()[1])
            os.environ["MASTER_ADDR"] = "127.0.0.1"
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl")
    c = CONFIGS["cfg4"]
    cap = (args.capacity or c["capacity"]) // world
    k = args.batch
    K = k * world
    cfg = P.RunConfig(batch_size=k, double=True, dueling=True, beta_end_step=50_000_000)
    on = P.build_network("atari", (84, 84, 4), 4, True)
    tg = P.build_network("atari", (84, 84, 4), 4, True)
    P.init_params(on, np.random.SeedSequence([1, 3]))          # identical on every rank
    P.sync_target(on, tg)
    opt = P.RmsProp(on, cfg.learning_rate, cfg.rms_decay, cfg.rms_epsilon)
    mem = P.PrioritizedReplay(cap, (84, 84, 4), P.PriorityConfig(0.6, 0.01, cfg.beta_schedule()),
                              shareable=True)
    mem.fill_synthetic(100 + rank, cap)
    learner = dp.DeviceDataParallelLearner(on, tg, mem, opt, cfg)
    rng = np.random.default_rng(np.random.SeedSequence([1, 2]))  # common draws on all ranks
    step0 = 50_000
    for s in range(args.warmup):
        learner.step(rng.random(K), mem.beta(step0 + s))
    assert learner.graph_exec is not None, "data-parallel graph was not captured"
    n0 = _lib.lib.dqn_launch_count()
    agent.USE_GRAPH = False
    g_saved = learner.graph_exec
    learner.graph_exec = None
    learner.step(rng.random(K), mem.beta(step0 + args.warmup))        # one eager step: count
    launches = int(_lib.lib.dqn_launch_count() - n0)
    learner.graph_exec = g_saved
    agent.USE_GRAPH = True

    # --- device-resident loop: pre-drawn inputs in HBM, one graph per update
    draws = np.empty((args.steps, K + 1))
    for s in range(args.steps):
        draws[s, :K] = rng.random(K)
        draws[s, K] = mem.beta(step0 + 200 + s)
    d_draws = torch.as_tensor(draws, device="cuda")
    slot = torch.zeros_like(d_draws[0])
    saved = learner.h_in
    learner.h_in = slot
    g_keep, g = agent.capture_graph(learner.enqueue, learner.plan.capture_stream)
    learner.h_in = saved
    sp = torch.cuda.current_stream().cuda_stream
    stream = torch.cuda.current_stream()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for s in range(args.steps):
            slot.copy_(d_draws[s], non_blocking=True)
            g.launch(sp)
            if (s + 1) % TARGET_SYNC_UPDATES == 0:
                P.sync_target(on, tg)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * args.steps / (ms / 1e3)

    # --- e2e: the public step() with host draws and host results
    dist.barrier()
    torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for s in range(args.steps):
        learner.step(rng.random(K), mem.beta(step0 + 400 + s))
    e3.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e2.elapsed_time(e3)], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e = world * args.steps / (float(t.item()) / 1e3)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT,
            "unit_note": "batch-32 learner updates/s summed over the GPUs (= global updates/s x N)",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hash-generated u8 frames per shard, random-init nets)",
            "config": bench_config("cfg4", cap * world, k, world, "dp"),
            "exchange": "sharded PER (shard totals all-gathered), frames read from the owners' "
                        "rings over NVLink (CUDA-IPC), NCCL gradient all-reduce",
            "transitions_per_sec": value * k,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * (K + 1),
                    "d2h_bytes_per_step": 8 * 4 * K + 4,
                    "path": "dp.DeviceDataParallelLearner.step (one graph launch per update)"},
            "gpu_launches": launches * args.steps, "launches_per_step": launches,
            "clocks": clk.summary(),
            "cpu_baseline": (cpu_baseline_obj("cfg4", k, 1 << 30, 2, args.cpu_budget,
                                              args.cpu_budget_1core)
                             if world == 1 and not args.no_cpu else None),
        }
        print(json.dumps(line), flush=True)
    learner.close()
    dist.destroy_process_group()


def resolve_mode(args, n_gpus: int) -> str:
    """N = 1: the single-GPU learner (cfg4); N > 1: the cfg5 data-parallel
    learner unless --mode replicas asks for the population of seeds."""
    if args.mode == "auto":
        return "single" if n_gpus == 1 else "dp"
    return args.mode


def spawn_ranks(n: int) -> int:
    """``python bench.py --gpus N`` outside torchrun: launch N ranks (one per
    GPU) through torch.distributed.run on this node and return its exit code.
    Refuses loudly when this box has fewer than N GPUs."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {n} requested but only {have} "
                          f"CUDA device(s) are visible; refusing to time fewer GPUs"}), flush=True)
        return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=sorted(CONFIGS))
    ap.add_argument("--capacity", type=int, default=0)
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-budget-1core", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "replicas", "dp"],
                    help="auto: N = 1 -> the single-GPU learner, N > 1 -> dp; dp: the cfg5 "
                         "data-parallel learner (sharded PER, NCCL gradient all-reduce); "
                         "replicas: one independent learner per GPU (population of seeds)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, _ = dist_env()
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if world > 1 and args.gpus not in (1, world):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    args.gpus = world
    if world > 1:
        # communicator set-up lines (ranks, NVLS / P2P transport) on stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,ENV")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    mode = resolve_mode(args, world)
    if mode == "dp":
        run_dp(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
