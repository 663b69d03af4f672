#!/usr/bin/env bash
# Run on the GPU box: the reference's own tests with its hot-path entry
# points bound to libbltc (tools/ref_suite/bltc_b200_substitute.py).
#   bash tools/ref_suite/run.sh [pytest args]      (BLTC_MODE=parity|strict|fast)
cd "$(dirname "$0")/../.."
export PYTHONPATH="$PWD/baseline/_ref:$PWD/tools/ref_suite:$PWD${PYTHONPATH:+:$PYTHONPATH}"
cd baseline/_ref/_tests
exec python -m pytest -p bltc_b200_substitute -p no:cacheprovider "$@"
