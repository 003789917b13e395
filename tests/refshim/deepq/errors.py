from paper_1804_05834_b200.errors import *  # noqa: F401,F403
