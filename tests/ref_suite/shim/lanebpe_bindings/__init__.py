"""Alias package: `import lanebpe_bindings` resolves to this package's
bindings module (TokenizerHandle).  Test infrastructure only."""

import sys

import lanebpe  # noqa: F401  (registers the lanebpe aliases first)
from paper_2603_02597_b200 import bindings as _bindings

sys.modules["lanebpe_bindings"] = _bindings
