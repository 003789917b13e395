"""Benchmark of the DQN learner update (BASELINE.json metric: learner
updates/s and sampled transitions/s, Dueling+Double+PER, batch 32, 1M
synthetic Atari transitions).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

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
             host's cores for a bounded sample.
``--impl reference`` times that CPU path alone and prints its own line.
Under torchrun (N > 1) the default is N independent learners, one per GPU
(the population-of-seeds mode: each rank owns its own 1M ring, tree and
networks; no data-path collective; weak scaling).  ``--mode dp`` runs the
cfg5 data-parallel learner instead (paper_1804_05834_b200/dp.py: replay
sharded across the ranks, global stratified PER over all-gathered shard
totals, per-GPU batch 32, NCCL gradient all-reduce; host-orchestrated, see
DESIGN.md §6).  Rank 0 reports the max-over-ranks time.
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
             "clocks_event_reasons.sw_power_cap")
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
        sm = sorted(float(r[0]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][1]), "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------------
# CPU side: the oracle port of the reference learn_step
# --------------------------------------------------------------------------

def cpu_learner(cfg_name: str, seed: int = 0, pool: int = 2048):
    """Oracle learner at the bench config.  The 1M-leaf fp64 tree is real; the
    frame store is a pool of ``pool`` synthetic transitions addressed by
    slot % pool (the reference's float32 ring would need 226 GB of host RAM;
    gather cost per sample is unchanged: one fancy-index copy per state)."""
    from oracle import deepq_oracle as O
    from paper_1804_05834_b200 import synth
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
    lcfg = O.LearnCfg(double=c["double"])
    return on, tg, mem, opt, lcfg, O


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [d.get("num_threads", 1) for d in threadpool_info() if d.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_time(cfg_name: str, steps: int, warmup: int, budget_s: float | None):
    """Time the oracle learn_step; returns (updates/s, steps timed)."""
    on, tg, mem, opt, lcfg, O = cpu_learner(cfg_name)
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


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    ups, n = cpu_time(args.config, args.steps, args.warmup, None)
    cores = blas_threads()
    sample = (f"{n} oracle learn_step updates ({args.config}, batch 32, 1M-leaf fp64 tree, "
              f"pooled frame store) after {args.warmup} warm-up, numpy/OpenBLAS {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": ups, "unit": UNIT, "n_gpus": args.gpus,
        "steps": n, "warmup": args.warmup, "ms_per_step": 1000.0 / ups, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": CONFIGS[args.config]["desc"], "global_batch": 32,
                   "parallelism": "host cpu"},
        "transitions_per_sec": ups * 32,
        "cpu_baseline": {"value": ups, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample, "cpu": cpu_model()},
        "e2e": {"value": ups, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
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
        ups, n = cpu_time(args.config, 1 << 30, 2, args.cpu_budget)
        cores = blas_threads()
        cpu = {"value": ups, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": (f"{n} oracle learn_step updates in ~{args.cpu_budget:.0f} s ({args.config}, "
                          f"batch 32, 1M-leaf fp64 tree, pooled frame store), numpy/OpenBLAS "
                          f"{cores} threads"),
               "cpu": cpu_model()}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hash-generated u8 84x84x4 frames, seeded metadata, random-init nets)",
            "config": {"workload": c["desc"], "capacity": cap, "global_batch": k * world,
                       "per_gpu_batch": k,
                       "parallelism": "single GPU" if world == 1 else f"replicas x{world}",
                       "l2": "inputs larger than L2 (56 GB u8 ring); parameters stay L2-resident "
                             "across updates as in training",
                       "fill_seconds": round(t_fill, 2)},
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
            "metric": METRIC, "value": value, "unit": UNIT + " (batch-32 updates, all GPUs)",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (hash-generated u8 frames per shard, random-init nets)",
            "config": {"workload": "cfg5 Dueling+Double+PER data-parallel, replay sharded",
                       "capacity": cap * world, "global_batch": K, "per_gpu_batch": k,
                       "parallelism": f"dp{world} (sharded PER, peer-ring gather, NCCL allreduce)",
                       "l2": "1M-slot ring (56 GB) >> L2: sampled rows come from HBM"},
            "transitions_per_sec": value * k,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": 8 * (K + 1),
                    "d2h_bytes_per_step": 8 * 4 * K + 4,
                    "path": "dp.DeviceDataParallelLearner.step (one graph launch per update)"},
            "gpu_launches": launches * args.steps, "launches_per_step": launches,
            "clocks": clk.summary(), "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    learner.close()
    dist.destroy_process_group()


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
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--mode", default="auto", choices=["auto", "single", "replicas", "dp"],
                    help="auto/replicas: one independent learner per GPU (population of "
                         "seeds; N = 1 is the single-GPU learner); dp: the cfg5 "
                         "data-parallel learner (sharded PER, NCCL gradient all-reduce)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = dist_env()[1]
    if args.impl == "reference":
        run_reference(args)
    elif args.mode == "dp":
        run_dp(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
