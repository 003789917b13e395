from paper_1804_05834_b200.config import RunConfig, resolve_config  # noqa: F401
