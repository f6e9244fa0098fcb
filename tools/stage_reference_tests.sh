#!/bin/bash
# Stage the reference's own test-suite (mipserve tests, /root/reference/pkg/tests)
# against THIS package, outside git: build/ref_tests/ (git-ignored; it travels
# to the GPU box with the gpurun snapshot).  A `mipserve` alias package maps
# every reference module name onto paper_1706_01449_b200's module of the same
# name, so the tests' imports and monkeypatches (e.g. opt.brute.measure_throughput)
# hit this implementation.  The service and CLI suites are out of scope.
#
#   bash tools/stage_reference_tests.sh            # here (needs /root/reference)
#   (cd build/ref_tests && PYTHONPATH=../..:. python -m pytest -q)   # on the GPU box
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg/tests
DST="$ROOT/build/ref_tests"
rm -rf "$DST"
mkdir -p "$DST/mipserve"
for t in conftest.py test_brute.py test_index.py test_clustering.py test_optimizer.py test_acceptance.py \
         test_model_io.py; do
  cp "$SRC/$t" "$DST/$t"
done
cat > "$DST/mipserve/__init__.py" <<'PY'
"""Alias of paper_1706_01449_b200 under the reference's package name (test staging only)."""
import sys as _sys

import paper_1706_01449_b200 as _pkg
from paper_1706_01449_b200 import *  # noqa: F401,F403
from paper_1706_01449_b200 import __all__  # noqa: F401

for _name in ("brute", "clustering", "index", "optimizer", "model_io"):
    _mod = __import__(f"paper_1706_01449_b200.{_name}", fromlist=[_name])
    _sys.modules[f"mipserve.{_name}"] = _mod
    globals()[_name] = _mod
__version__ = getattr(_pkg, "__version__", "0.1.0")
PY
cat > "$DST/pytest.ini" <<'INI'
[pytest]
addopts = -p no:cacheprovider
INI
echo "staged $(ls "$DST"/test_*.py | wc -l) reference test files into $DST"
