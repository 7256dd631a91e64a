#!/bin/bash
# One gpurun call for a round checkpoint: build, the GPU test suite, the default bench line (config
# 2 + every other BASELINE config), the launch list of the bench command, and ncu --set full of the
# solver kernel per config (caches flushed between replays, and warm for the listed configs).
# usage (under gpurun): bash tools/gpu_round.sh TAG [TESTS=1] [NCU_CFGS="1 2 3 4 5"] [WARM_CFGS="2 3 4"]
TAG=${1:-r2}
TESTS=${2:-1}
NCU_CFGS=${3:-"1 2 3 4 5"}
WARM_CFGS=${4:-"2 3 4"}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { cat gpurun_out/${TAG}_build.log; exit 1; }
if [ "$TESTS" = "1" ]; then
  timeout 2700 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${TAG}_gpu_tests.log 2>&1
  echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_gpu_tests.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --other-configs "" --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/${TAG}_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --other-configs "" --no-cpu-baseline --steps 2 --warmup 3 --e2e-steps 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
for c in $NCU_CFGS; do
  timeout 300 python tools/prof.py $c 30 > gpurun_out/${TAG}_prof_cfg$c.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ajm_(solve|band|resident)_kernel" -s 1 -c 1 \
      -o gpurun_out/${TAG}_ncu_cfg$c -f python tools/prof.py $c 30 > gpurun_out/${TAG}_ncu_cfg$c.log 2>&1
  echo "ncu cfg$c rc=$?"
done
for c in $WARM_CFGS; do
  timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"ajm_(solve|band|resident)_kernel" -s 1 -c 1 \
      -o gpurun_out/${TAG}_ncuwarm_cfg$c -f python tools/prof.py $c 30 > gpurun_out/${TAG}_ncuwarm_cfg$c.log 2>&1
  echo "ncu warm cfg$c rc=$?"
done
# gpurun brings back <= 64 MiB: export the raw / source pages as CSV here and drop the reports
for r in gpurun_out/${TAG}_ncu*_cfg*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page source --csv > "${r%.ncu-rep}.source.csv" 2>/dev/null
  gzip -f "${r%.ncu-rep}.source.csv"
  rm -f "$r"
done
du -sh gpurun_out
ls gpurun_out | grep "^${TAG}_" | head -60
