#!/bin/bash
# One gpurun call for a development checkpoint: build, selected GPU tests, A/B timing against a
# reference library (abtest/<REF>.so from tools/ab_build.sh).
# usage (under gpurun): bash tools/gpu_check.sh TAG "PYTEST_ARGS" REF CFGS
TAG=${1:-chk}; PT=${2:-"tests -m gpu -x -q"}; REF=${3:-}; CFGS=${4:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail -30 gpurun_out/${TAG}_build.log; exit 1; }
if [ -n "$PT" ]; then
  timeout 1500 python -m pytest $PT > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/${TAG}_tests.log
fi
if [ -n "$REF" ]; then
  timeout 1500 bash tools/ab.sh $REF $CFGS > gpurun_out/${TAG}_ab.log 2>&1; echo "ab rc=$?"; cat gpurun_out/${TAG}_ab.log
fi
