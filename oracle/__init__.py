"""CPU oracle for the in-GPU experience-replay DQN train step (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1801_03138_b200`` never imports it.  See ``oracle/oracle.c`` for the arithmetic
and its citations.
"""
from .oracle import *  # noqa: F401,F403
