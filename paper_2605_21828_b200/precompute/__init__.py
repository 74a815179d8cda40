"""Host precompute: trees, interpolative decompositions, plan writer.

Outside the timed hot path (BASELINE.json north_star: "Factorization
construction ... is a host precompute outside the timed path").
"""
from .builder import build_plan  # noqa: F401
from .planfile import PlanView, PlanWriter  # noqa: F401
from .trees import freq_tree, kd_tree  # noqa: F401
