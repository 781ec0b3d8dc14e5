"""Alias package: `import lanebpe` resolves to paper_2603_02597_b200 so the
reference's own test suite (tests/ref_suite/_vendor) runs against this
package unchanged.  Test infrastructure only.

Submodules are registered under the reference's module names so that
`from lanebpe.merge_table import ...`, `from lanebpe import chunker` and the
exception classes are the very objects this package uses (no second import
of any module).  `lanebpe.bench` gathers the reference bench module's names
(windows.py + report.py); `lanebpe.cli` is a stub: the CLI is out of scope
(DESIGN.md section 7), so the tests that drive it fail by design.
"""

import sys
import types

import paper_2603_02597_b200 as _pkg
from paper_2603_02597_b200 import bindings, byte_codec, chunker, engine, errors, merge_table, report, windows

_bench = types.ModuleType("lanebpe.bench", "reference bench.py names: windows.py + report.py")
for _mod in (windows, report):
    for _k, _v in vars(_mod).items():
        if not _k.startswith("__"):
            setattr(_bench, _k, _v)

_cli = types.ModuleType("lanebpe.cli", "stub: the lanebpe CLI is out of scope for this package")


def _no_cli(argv=None):
    raise NotImplementedError("the lanebpe CLI (cli.py) is out of scope for the B200 encoder")


_cli.main = _no_cli

for _name, _mod in {"errors": errors, "merge_table": merge_table, "chunker": chunker, "engines": engine,
                    "byte_codec": byte_codec, "bench": _bench, "cli": _cli, "bindings": bindings}.items():
    sys.modules[f"lanebpe.{_name}"] = _mod
    setattr(_pkg, _name, _mod)
sys.modules["lanebpe"] = _pkg
