from paper_1804_05834_b200.schedules import LinearSchedule  # noqa: F401
