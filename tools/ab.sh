#!/bin/bash
# A/B under gpurun: the current build vs a reference library (abtest/<ref>.so, built from a commit
# with tools/ab_build.sh), same box, interleaved, 2 rounds.
# usage: bash tools/ab.sh REF CFGS [L2MODES]      e.g. bash tools/ab.sh libajm_2b49c86 2,5 3
REF=$1; CFGS=${2:-2}; L2=${3:-3}
python -c "import __graft_entry__ as g; g.build()" || exit 1
for i in 1 2; do
  AJM_LIB_OVERRIDE=$PWD/abtest/$REF.so timeout 600 python tools/quick.py $CFGS 0 $L2 0 2>&1 | grep "500its\|^cfg" | sed "s/^/ref  /"
  timeout 600 python tools/quick.py $CFGS 0 $L2 0 2>&1 | grep "500its\|^cfg" | sed "s/^/curr /"
done | sed 's/n=.*//' | paste - - | awk '{print $1,$2,$3,$4,$8}'
