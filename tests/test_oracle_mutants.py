"""Mutation harness for the oracle pins (seven CC1 / CC2-avg misreadings
survived every pin).  Each mutant in tests/oracle_mutants.py is loaded in place of
oracle/oracle.py and the whole pin suite (tests/test_oracle_pins.py) runs against
it in a subprocess; the suite must fail (pytest exit status 1) for every mutant.
CPU only; the subprocesses run in parallel."""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import oracle_mutants  # noqa: E402

ROOT = os.path.dirname(HERE)


def _run(name):
    env = dict(os.environ, HM_ORACLE_MUTANT=name, OMP_NUM_THREADS="1")
    p = subprocess.run([sys.executable, "-m", "pytest", os.path.join(HERE, "test_oracle_pins.py"),
                        "-x", "-q", "-p", "no:cacheprovider", "-p", "no:randomly"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    return name, p.returncode, p.stdout[-2000:]


def test_every_mutant_applies():
    for name, *_ in oracle_mutants.MUTANTS:
        src = oracle_mutants.mutated_source(name)       # raises unless the fragment occurs once
        assert src != open(oracle_mutants.ORACLE_SRC).read()


def test_pins_kill_every_mutant():
    names = [m[0] for m in oracle_mutants.MUTANTS]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(_run, names))
    survivors = [(n, rc, out) for n, rc, out in results if rc != 1]
    assert not survivors, "\n\n".join(f"{n}: exit {rc}\n{out}" for n, rc, out in survivors)
