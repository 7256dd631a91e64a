#!/bin/bash
# A/B under gpurun of whole library builds: the current build vs abtest/<REF>.so (tools/ab_build.sh),
# separate processes, interleaved, ROUNDS rounds (tools/env_ab.py timing: 3 solves after a warm-up).
# usage: bash tools/lib_ab.sh REF CFGS [ROUNDS] [ENV]     e.g. bash tools/lib_ab.sh libajm_0f91b5b 2,5 2
REF=$1; CFGS=${2:-2}; ROUNDS=${3:-2}; ENVV=${4:-}
for i in $(seq $ROUNDS); do
  AB_ROUNDS=1 AJM_LIB_OVERRIDE=$PWD/abtest/$REF.so timeout 900 python tools/env_ab.py $CFGS "$ENVV" 2>&1 | grep "^cfg" | sed "s/^/ref  /"
  AB_ROUNDS=1 timeout 900 python tools/env_ab.py $CFGS "$ENVV" 2>&1 | grep "^cfg" | sed "s/^/curr /"
done
