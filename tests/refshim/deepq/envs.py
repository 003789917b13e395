from paper_1804_05834_b200.envs import *  # noqa: F401,F403
from paper_1804_05834_b200.envs import Catch, GridWorld, TabularChain, make_env  # noqa: F401
