#!/bin/bash
# One gpurun call: bench line for every BASELINE config, then an ncu --set full capture of the
# solver kernel (2nd launch of tools/prof.py = a 31-pass solve) per config.
# usage (under gpurun): bash tools/gpu_configs.sh "1 3 4 5" [tag]
CFGS=${1:-"1 2 3 4 5"}
TAG=${2:-r1}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for c in $CFGS; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_bench_cfg$c.json 2> gpurun_out/${TAG}_bench_cfg$c.err
done
for c in $CFGS; do
  python tools/prof.py $c 30 > gpurun_out/${TAG}_prof_cfg$c.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"ajm_(solve|band|resident)_kernel" -s 1 -c 1 \
      -o gpurun_out/${TAG}_ncu_cfg$c -f python tools/prof.py $c 30 > gpurun_out/${TAG}_ncu_cfg$c.log 2>&1
done
ls -la gpurun_out
