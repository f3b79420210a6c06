#!/bin/bash
# GPU box: the reference's tests/test_subdivision.py, test_cache.py and test_renderer.py with
# the record path rebound to the device engine (tools/rebind_plugin.py).  Summary line and
# per-test outcomes → gpurun_out/ref_tests_rebound.log
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
cd "$ROOT/baseline/_ref/ref_pkg/tests" || { echo "baseline/_ref not staged (tools/stage_reference.sh)"; exit 1; }
PYTHONPATH="$ROOT/baseline/_ref:$ROOT:$ROOT/tools" PYTHONDONTWRITEBYTECODE=1 timeout 3000 \
  python -m pytest -p rebind_plugin -p no:cacheprovider test_subdivision.py test_cache.py test_renderer.py \
  -q -rA "$@" > "$ROOT/gpurun_out/ref_tests_rebound.log" 2>&1
echo "rc=$?" >> "$ROOT/gpurun_out/ref_tests_rebound.log"
tail -5 "$ROOT/gpurun_out/ref_tests_rebound.log"
