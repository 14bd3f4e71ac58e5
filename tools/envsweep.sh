#!/bin/bash
# Runtime-knob sweep (no rebuild): tools/envsweep.sh "c2 c2d" "GC3_UNIT_WARPS=2 GC3_TMA=0;GC3_LANES=5" [bench args]
configs=$1
IFS=';' read -ra sets <<< "$2"
extra=${3:-}
for s in "${sets[@]}"; do
  for c in $configs; do
    r=$(env $s timeout 120 python bench.py --config $c --quick --steps 20 $extra 2>&1 | tail -1)
    echo "[$s] $c $r"
  done
done
