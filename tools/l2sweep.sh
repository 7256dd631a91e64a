#!/bin/bash
# L2 policy sweep, every case in a FRESH process (persisting L2 lines survive a handle and bias
# the next one in the same process)
CFG=${1:-2}
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
for case in "auto:" "m2:AJM_L2MODE=2" "m3:AJM_L2MODE=3" "np2:AJM_L2PERSIST=0 AJM_L2MODE=2" "np3:AJM_L2PERSIST=0 AJM_L2MODE=3" "np0:AJM_L2PERSIST=0 AJM_L2MODE=0"; do
  name=${case%%:*}; envs=${case#*:}
  for rep in 1 2; do
    env $envs timeout 300 python tools/quick.py $CFG 0 -1 0 2>&1 | grep "500its" | sed "s/^/$name /"
  done
done
