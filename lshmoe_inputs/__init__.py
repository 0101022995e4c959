"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

This module holds none of the method's arithmetic (no hashing, bucketing, centroid, expert or
restore step): it only draws tokens, gate assignments, expert weights and the rotation seed.
"""
from .gen import *  # noqa: F401,F403
