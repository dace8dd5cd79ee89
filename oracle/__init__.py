"""ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports it.
"""
from .oracle import *  # noqa: F401,F403
from . import oracle as core  # noqa: F401
from ._bfs import build, num_threads  # noqa: F401
