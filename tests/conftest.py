"""Shared fixtures.  `gpu` marks tests that need a B200 (run with -m gpu)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle

    oracle.build()
    return oracle


@pytest.fixture(scope="session")
def cpg():
    import paper_2412_10789_b200 as P

    return P


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu():
    if not has_gpu():
        pytest.skip("no CUDA device")
    return 0


# Tolerances of the north star: per score vector, max-abs 1e-12 and L1 1e-10,
# identical top-100 set (value desc, id asc) -- up to structural ties: nodes whose
# scores are within 1e-12 of the 100th score in both vectors may swap in or out
# (equal reference scores broken by last-bit rounding, e.g. symmetric rings).
MAX_ABS = 1e-12
L1 = 1e-10


def assert_parity(got, ref, topk=100, max_abs=MAX_ABS, l1=L1):
    from oracle import parity

    p = parity(got, ref, topk)
    assert p["max_abs"] <= max_abs, p
    assert p["l1"] <= l1, p
    assert p["topk_equal_mod_ties"], p
    return p
