"""Golden fixtures for the acting side, generated
from the UNMODIFIED reference in the build container:

    python tests/golden/make_trainer_golden.py

* envs.npz         frame / reward / terminal sequences of Catch, GridWorld and
                   TabularChain under seeded random actions; preprocess_frame
                   and Preprocessor outputs (envs.py:61-357)
* trainer_catch.npz  the metric records of a short desk-preset Catch run of
                   the reference Trainer (agent.py:159-405), plus the norms
                   of its online parameters at the end
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from deepq.agent import Trainer  # noqa: E402
from deepq.config import resolve_config  # noqa: E402
from deepq.envs import Preprocessor, make_env, preprocess_frame  # noqa: E402
from deepq.metrics import RecordCollector  # noqa: E402

ENV_CASES = [
    ("catch", {}, 11),
    ("catch", {"height": 10, "width": 7, "paddle_width": 2}, 12),
    ("gridworld", {"size": 5, "max_steps": 30}, 13),
    ("tabular", {}, 14),
]

TRAINER_OVERRIDES = dict(preset="desk", env="catch", seed=5, max_steps=3000, learning_start=500,
                         test_period=1500, test_episodes=10, eps_end_step=2000, target_sync=500,
                         replay_capacity=2000)


def env_cases():
    out = {}
    for ci, (name, params, seed) in enumerate(ENV_CASES):
        env = make_env(name, rng=np.random.default_rng(seed), **params)
        arng = np.random.default_rng(100 + ci)
        frames, rewards, terms, acts = [env.reset()], [], [], []
        for _ in range(300):
            a = int(arng.integers(0, env.spec.n_actions))
            r = env.step(a)
            acts.append(a)
            frames.append(r.observation)
            rewards.append(r.reward)
            terms.append(r.terminal)
            if r.terminal:
                frames.append(env.reset())
        out[f"env{ci}_frames"] = np.stack(frames)
        out[f"env{ci}_actions"] = np.array(acts, dtype=np.int64)
        out[f"env{ci}_rewards"] = np.array(rewards, dtype=np.float64)
        out[f"env{ci}_terminals"] = np.array(terms, dtype=bool)
    rng = np.random.default_rng(7)
    cases = [((30, 40, 3), (24, 24)), ((210, 160, 3), (84, 84)), ((10, 7), (24, 24)),
             ((8, 8), (24, 24)), ((24, 24), (24, 24)), ((40, 30, 1), (17, 23))]
    for i, (shape, size) in enumerate(cases):
        f = rng.integers(0, 256, size=shape, dtype=np.uint8)
        out[f"pre{i}_in"] = f
        out[f"pre{i}_size"] = np.array(size)
        out[f"pre{i}_out"] = preprocess_frame(f, size)
    ff = rng.random((12, 9))
    out["pref_in"] = ff
    out["pref_out"] = preprocess_frame(ff, (5, 6))
    pre = Preprocessor((6, 5), 3)
    seq = [rng.integers(0, 256, size=(9, 8), dtype=np.uint8) for _ in range(6)]
    stacks = [pre.reset(seq[0])] + [pre.push(s) for s in seq[1:]]
    out["stack_in"] = np.stack(seq)
    out["stack_out"] = np.stack(stacks)
    return out


def trainer_case():
    cfg = resolve_config(TRAINER_OVERRIDES)
    sink = RecordCollector()
    t0 = time.time()
    tr = Trainer(cfg, sink=sink)
    tr.run()
    rows = []
    for r in sink.records:
        rows.append([r.step, -1 if r.episode is None else r.episode,
                     np.nan if r.episode_return is None else r.episode_return,
                     np.nan if r.epsilon is None else r.epsilon,
                     np.nan if r.beta is None else r.beta,
                     np.nan if r.mean_abs_td is None else r.mean_abs_td,
                     np.nan if r.loss is None else r.loss,
                     np.nan if r.eval_mean is None else r.eval_mean])
    out = {"records": np.array(rows, dtype=np.float64),
           "learn_steps": np.int64(tr.learn_steps),
           "elapsed_s": np.float64(time.time() - t0),
           "overrides": np.array(repr(TRAINER_OVERRIDES))}
    for n, t in tr.online.named_tensors():
        out[f"norm_{n}"] = np.float64(np.linalg.norm(t.values.astype(np.float64)))
    return out


if __name__ == "__main__":
    np.savez_compressed(HERE / "envs.npz", **env_cases())
    tc = trainer_case()
    print(f"reference trainer: {tc['records'].shape[0]} records, {int(tc['learn_steps'])} learn "
          f"steps, {float(tc['elapsed_s']):.1f} s")
    np.savez_compressed(HERE / "trainer_catch.npz", **tc)
