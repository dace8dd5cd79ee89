"""Seeded synthetic HoMLN inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the paper's method (no BFS, no closeness,
no aggregation, no composition).  It only draws edge lists from counter-based
SplitMix64 streams, so the oracle (``oracle/``) and the product
(``paper_2207_11662_b200``) can be fed byte-identical inputs without sharing
any code path of the method itself.

The recipes stand in for the paper's PaRMAT / RMAT data sets
(PAPER.md:770-775 §6, :821-822, :1295-1303 appendix), which are not
available here; the five configurations are those of ``BASELINE.json``.
"""
from .prng import Stream, stream_key, mix64  # noqa: F401
from .gen import (  # noqa: F401
    HoMLN, er_candidates, rmat_candidates, sbm_candidates, draw_unique_edges,
    keep_bernoulli, random_graph, build_config, CONFIG_NAMES,
)
