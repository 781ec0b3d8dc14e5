import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT, ROOT / "tools"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))

import fixtures  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def gpt2_paths():
    return fixtures.gpt2_paths()


@pytest.fixture(scope="session")
def oracle_tables(gpt2_paths):
    from oracle.oracle import load_tables

    return load_tables(*gpt2_paths)


@pytest.fixture(scope="session")
def oracle(oracle_tables):
    from oracle.oracle import OracleEncoder

    return OracleEncoder.from_tables(oracle_tables)


@pytest.fixture(scope="session")
def tokenizer(gpt2_paths):
    import paper_2603_02597_b200 as bpe

    return bpe.Tokenizer.from_files(*gpt2_paths)


@pytest.fixture(scope="session")
def prose_samples():
    return fixtures.prose_samples()


# the vendored reference suite runs in its own pytest process (test_ref_suite.py)
collect_ignore = ["ref_suite"]
