#!/bin/bash
# fresh-process timing of configs under env settings: bash tools/l2fresh.sh CFG "name:ENV=.. ENV2=.." ...
CFG=$1; shift
python -c "import __graft_entry__ as g; g.build()" >/dev/null || exit 1
for case in "$@"; do
  name=${case%%:*}; envs=${case#*:}
  for rep in 1 2; do env $envs timeout 300 python tools/quick.py $CFG 0 -1 0 2>&1 | grep "500its" | sed "s/^/$name /"; done
done
