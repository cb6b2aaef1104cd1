"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NONE of the method's arithmetic: the five BASELINE.json workload presets
(plain data), seeded trigonometric-polynomial black boxes (the synthetic functions the method
is run on, Thm 1.1), and seeded parameter points.  Both the product path and the
oracle may consume it; neither side's arithmetic lives here.
"""
from .configs import CONFIGS, EXAMPLES, config  # noqa: F401
from .fixtures import TrigPoly, trig_poly, uniform_points  # noqa: F401
