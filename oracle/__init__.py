"""LSH-MoE CPU oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference`` arm) may import, call or execute anything under ``oracle/``.  The product
path (``paper_2411_08446_b200``) never imports it and shares no code with it.

See ``oracle/lshmoe_oracle.py`` for the step-by-step implementation of the paper's Algorithm 1
(App. A) and ``oracle/brute.py`` for the pure-Python brute-force variants used
to pin the NumPy oracle on tiny inputs.
"""
from .lshmoe_oracle import *  # noqa: F401,F403
