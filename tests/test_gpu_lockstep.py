"""100-step parity of the device learner against the CPU oracle
(the protocol that replaces north_star's "1e-2 after
100 steps"; reference: agent.py:91-132, the reference's own 100-step case
test_agent.py:286-294).

* Teacher-forced lockstep, cfg1-cfg4 with Huber off and on: before every
  step the oracle's weights, RMSprop accumulators, tree and max priority are
  copied into the device learner, both take one update with the same draws,
  and the TD errors and every weight tensor must agree norm-wise within 1e-3
  at EVERY one of the 100 steps (target networks re-synced every 25 steps on
  both sides).
* Free-running drift: device and oracle run 100 updates from the same state
  with the same uniforms, never re-synced.  Reported next to the fp32
  re-ordering floor (the oracle against itself with the batch rows permuted,
  i.e. the same arithmetic summed in another order), as App. A.3 step 3
  prescribes; asserted only finite, not at 1e-2 (App. A.2: any re-associated
  fp32 learner drifts ~1e-1 from the reference by step 30).

Set DQN_PARITY_REPORT=<dir> to write the per-step curves as JSON.
"""

from __future__ import annotations

import json
import os
from pathlib import Path

import numpy as np
import pytest

from oracle import deepq_oracle as O
from tests.helpers import oracle_learner, rel_norm
from tests.test_gpu_learner import device_learner, teacher_force

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

TOL = 1e-3
STEPS = 100
SYNC_EVERY = 25
CAP = 128

CASES = {
    "cfg1": dict(dueling=False, double=False, per=False),
    "cfg1_huber": dict(dueling=False, double=False, per=False, huber=True),
    "cfg2": dict(dueling=False, double=True, per=False),
    "cfg2_huber": dict(dueling=False, double=True, per=False, huber=True),
    "cfg3": dict(dueling=False, double=True, per=True),
    "cfg3_huber": dict(dueling=False, double=True, per=True, huber=True),
    "cfg4": dict(dueling=True, double=True, per=True),
    "cfg4_huber": dict(dueling=True, double=True, per=True, huber=True),
}


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1804_05834_b200 as P
    return P


def _report(name: str, payload: dict) -> None:
    d = os.environ.get("DQN_PARITY_REPORT")
    if d:
        Path(d).mkdir(parents=True, exist_ok=True)
        (Path(d) / f"{name}.json").write_text(json.dumps(payload, indent=1))


def _weights_worst(on, o_params):
    errs = {n: rel_norm(t.values.cpu().numpy(), o_params[n]) for n, t in on.named_tensors()}
    w = max(errs, key=errs.get)
    return w, errs[w]


def _draws(st):
    return np.random.default_rng(900 + st)


@pytest.mark.parametrize("name", list(CASES))
def test_teacher_forced_lockstep_100(P, name):
    kw = CASES[name]
    on, tg, mem, opt, cfg = device_learner(P, cap=CAP, **kw)
    o_on, o_tg, o_mem, o_opt, o_cfg = oracle_learner(cap=CAP, **kw)
    rows = []
    for st in range(STEPS):
        teacher_force(P, on, tg, mem, opt, o_on, o_tg, o_mem, o_opt)
        step = 100 + 4 * st
        res = P.learn_step(on, tg, mem, opt, cfg, step, _draws(st))
        ores = O.learn_step(o_on, o_tg, o_mem, o_opt, o_cfg, step, rng=_draws(st))
        td = rel_norm(res.td_errors, ores["td_errors"])
        loss = rel_norm(res.losses, ores["losses"])
        wname, w = _weights_worst(on, o_on.params)
        rows.append({"step": st, "td": td, "loss": loss, "worst_tensor": wname, "worst_weight": w})
        assert td < TOL and loss < TOL, (st, td, loss)
        assert w < TOL, (st, wname, w)
        if kw["per"]:
            tree = rel_norm(mem.tree.nodes.cpu().numpy(), o_mem.tree.nodes)
            rows[-1]["tree"] = tree
            assert tree < 1e-5, (st, tree)
        if (st + 1) % SYNC_EVERY == 0:
            o_tg.copy_from(o_on)          # the device target is re-forced next step
    worst = max(r["worst_weight"] for r in rows)
    worst_td = max(r["td"] for r in rows)
    print(f"{name}: {STEPS} teacher-forced steps, worst weight rel-norm {worst:.2e}, "
          f"worst TD rel-norm {worst_td:.2e}")
    _report(f"lockstep_{name}", {"case": name, "steps": STEPS, "tol": TOL, "worst_weight": worst,
                                 "worst_td": worst_td, "rows": rows})


class _PermutedPer(O.PerReplay):
    """Oracle PER whose sampled batch comes back with its rows permuted: the
    same update summed in another order (the fp32 re-ordering floor)."""

    perm = None

    def sample(self, k, beta, rng=None, u=None):
        b = super().sample(k, beta, rng=rng, u=u)
        p = self.perm
        return O.Batch(b.states[p], b.actions[p], b.rewards[p], b.next_states[p], b.terminals[p],
                       b.indices[p], b.probabilities[p], b.weights[p])


def test_free_running_drift_curve(P):
    """cfg4, 100 free-running updates: device vs oracle next to the oracle vs
    its row-permuted self.  Reported (DQN_PARITY_REPORT), asserted finite and
    the first step within 1e-3."""
    kw = CASES["cfg4"]
    on, tg, mem, opt, cfg = device_learner(P, cap=CAP, **kw)
    o_on, o_tg, o_mem, o_opt, o_cfg = oracle_learner(cap=CAP, **kw)
    f_on, f_tg, f_mem, f_opt, _ = oracle_learner(cap=CAP, **kw)
    pm = _PermutedPer.__new__(_PermutedPer)
    pm.__dict__.update(f_mem.__dict__)
    pm.perm = np.random.default_rng(5).permutation(32)
    teacher_force(P, on, tg, mem, opt, o_on, o_tg, o_mem, o_opt)
    rows = []
    for st in range(STEPS):
        step = 100 + 4 * st
        P.learn_step(on, tg, mem, opt, cfg, step, _draws(st))
        O.learn_step(o_on, o_tg, o_mem, o_opt, o_cfg, step, rng=_draws(st))
        O.learn_step(f_on, f_tg, pm, f_opt, o_cfg, step, rng=_draws(st))
        _, dev = _weights_worst(on, o_on.params)
        floor = max(rel_norm(f_on.params[n], o_on.params[n]) for n in o_on.params)
        fc1 = rel_norm(dict(on.named_tensors())["fc1.weight"].values.cpu().numpy(),
                       o_on.params["fc1.weight"])
        rows.append({"step": st + 1, "device_vs_oracle": dev, "fc1_weight": fc1,
                     "reorder_floor": floor})
        assert np.isfinite(dev)
        if (st + 1) % SYNC_EVERY == 0:
            P.sync_target(on, tg)
            o_tg.copy_from(o_on)
            f_tg.copy_from(f_on)
    assert rows[0]["device_vs_oracle"] < TOL
    pick = [r for r in rows if r["step"] in (1, 10, 30, 100)]
    print("drift: " + "  ".join(f"step {r['step']}: dev {r['device_vs_oracle']:.1e} "
                                f"floor {r['reorder_floor']:.1e}" for r in pick))
    _report("drift_cfg4", {"case": "cfg4", "steps": STEPS, "rows": rows})
