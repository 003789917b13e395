"""deepq.agent over the device learner."""

from __future__ import annotations

import paper_1804_05834_b200 as P

from ._host import to_np
from .network import Network, unwrap
from .replay import unwrap_memory


def learn_step(online, target, memory, optimizer, config, step, rng):
    opt = optimizer._opt if hasattr(optimizer, "_opt") else optimizer
    return P.learn_step(unwrap(online), unwrap(target), unwrap_memory(memory), opt, config, step, rng)


def compute_target_dqn(batch, target_net, gamma):
    return to_np(P.compute_target_dqn(batch, unwrap(target_net), gamma))


def compute_target_double(batch, online_net, target_net, gamma):
    return to_np(P.compute_target_double(batch, unwrap(online_net), unwrap(target_net), gamma))


def select_action(net, state, eps, rng):
    return P.select_action(unwrap(net), state, eps, rng)


def evaluate(net, env, episodes, test_eps, rng, *args, **kwargs):
    return P.evaluate(unwrap(net), env, episodes, test_eps, rng, *args, **kwargs)


def anneal_epsilon(step, schedule):
    return P.trainer.anneal_epsilon(step, schedule)


__all__ = ["learn_step", "compute_target_dqn", "compute_target_double", "select_action",
           "evaluate", "anneal_epsilon", "Network"]
