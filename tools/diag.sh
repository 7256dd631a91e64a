#!/bin/bash
# Diagnostics of the current build under gpurun: per-pass phase split (AJM_TS) and an ncu --set full
# capture (warm L2, source page exported) of the solver kernel, per config.
# usage: bash tools/diag.sh TAG "CFGS" [PASSES]
TAG=${1:-d}; CFGS=${2:-2}; P=${3:-30}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
for c in $CFGS; do
  AJM_TS=1 timeout 300 python tools/prof.py $c $P 2>&1 | grep -v "^\[ajm create\]" | tail -4
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"ajm_(solve|band|resident)_kernel" -s 1 -c 1 \
      -o gpurun_out/${TAG}_cfg$c -f python tools/prof.py $c $P > gpurun_out/${TAG}_ncu_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?"
  r=gpurun_out/${TAG}_cfg$c.ncu-rep
  ncu -i $r --page raw --csv > gpurun_out/${TAG}_cfg$c.raw.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source cuda,sass > gpurun_out/${TAG}_cfg$c.src.csv 2>/dev/null
  ncu -i $r --page source --csv > gpurun_out/${TAG}_cfg$c.source.csv 2>/dev/null
  python tools/ncu_src.py gpurun_out/${TAG}_cfg$c.source.csv 2>&1 | head -30
  gzip -f gpurun_out/${TAG}_cfg$c.src.csv gpurun_out/${TAG}_cfg$c.source.csv
  rm -f $r
done
