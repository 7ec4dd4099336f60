"""synth/ -- seeded synthetic input generators shared by tests, bench and the
oracle legs.  Holds no arithmetic of the EAT method (see timetable.py)."""
from .timetable import CONFIGS, SINGLE_QUERY, Timetable, generate, queries, random_small, stats  # noqa: F401
