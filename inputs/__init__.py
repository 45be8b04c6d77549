"""Seeded synthetic input generators shared by the tests, the bench and smoke().

This module holds none of the method's arithmetic: it only draws experiences and
initial parameter blobs from seeded numpy Philox streams (recipe in DESIGN.md
"Synthetic inputs").  Both the CUDA path and the oracle consume what it returns.
"""
from .synth import *  # noqa: F401,F403
