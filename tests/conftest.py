import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

# Mutation testing of the oracle pins (tests/test_oracle_mutants.py): run the pin
# suite against a deliberately broken oracle; it must fail.
if os.environ.get("HM_ORACLE_MUTANT"):
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import oracle_mutants
    oracle_mutants.install(os.environ["HM_ORACLE_MUTANT"])


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def pytest_collection_modifyitems(config, items):
    # -m gpu selects GPU tests; without a device they fail loudly instead of
    # silently passing on a fallback (there is none).
    pass


@pytest.fixture(scope="session")
def root():
    return ROOT
