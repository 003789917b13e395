"""Import-alias shim: the reference package name ``deepq`` over the device
package ``paper_1804_05834_b200``, so that the reference's own unit tests
(pkg/tests/test_replay.py, test_optim.py, test_agent.py) run UNCHANGED
against the B200 implementation (tools/run_reference_suite.py).

Adaptations, all at the API boundary (no computation here):
* device tensors are exposed as numpy arrays / live host views (_host.py);
* float64 networks / rings, which the reference supports and the device
  learner does not (it computes in fp32 and raises ConfigError), are built
  as float32 -- the tests that depend on float64 accuracy (rtol 1e-9 and
  below, finite differences) are expected to fail and are listed as such.
"""

from .agent import (anneal_epsilon, compute_target_double, compute_target_dqn,  # noqa: F401
                    evaluate, learn_step, select_action)
from .config import RunConfig  # noqa: F401
from .network import Network, build_network, init_params  # noqa: F401
from .optim import RmsProp, clip_gradients, sync_target  # noqa: F401
from .replay import (PrioritizedReplay, PriorityConfig, ReplayMemory,  # noqa: F401
                     SampleBatch, SumTree, Transition, anneal_beta)
from .schedules import LinearSchedule  # noqa: F401
