#!/usr/bin/env python3
"""Copy the reference's own test suite into tests/ref_suite/_vendor/ (test
infrastructure only, git-ignored: never part of the product or the history).

    python tests/ref_suite/sync.py [/root/reference/pkg]

Layout mirrors the reference package so its conftest paths resolve:
  _vendor/tests/           <- pkg/tests            (unit, property, acceptance)
  _vendor/bindings/tests/  <- pkg/bindings/tests   (TokenizerHandle contract)
tests/test_ref_suite.py then runs that suite against this package through the
`lanebpe` / `lanebpe_bindings` alias packages in tests/ref_suite/shim/.
The copy travels to the GPU box with the working tree (gpurun snapshots it);
/root/reference itself does not.
"""

from __future__ import annotations

import shutil
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
VENDOR = HERE / "_vendor"


def sync(pkg: Path) -> None:
    if not (pkg / "tests").is_dir():
        raise SystemExit(f"{pkg}/tests not found")
    if VENDOR.exists():
        shutil.rmtree(VENDOR)
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache", ".hypothesis")
    shutil.copytree(pkg / "tests", VENDOR / "tests", ignore=ignore)
    shutil.copytree(pkg / "bindings" / "tests", VENDOR / "bindings" / "tests", ignore=ignore)
    n = sum(1 for _ in VENDOR.rglob("test_*.py"))
    print(f"synced {n} test modules from {pkg} into {VENDOR}")


if __name__ == "__main__":
    sync(Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg"))
