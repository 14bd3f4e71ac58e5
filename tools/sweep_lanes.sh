#!/bin/bash
# lanes x tile sweep per config (no rebuild): tools/sweep_lanes.sh "c2:9,12,18:16384,32768,65536" ...
for spec in "$@"; do
  c=${spec%%:*}; rest=${spec#*:}; lanes=${rest%%:*}; tiles=${rest#*:}
  for l in ${lanes//,/ }; do for t in ${tiles//,/ }; do
    r=$(GC3_MAX_LANES=64 timeout 100 python bench.py --config $c --quick --steps 10 --lanes $l --tile-bytes $t 2>&1 | tail -1)
    echo "$c lanes=$l tile=$t $r"
  done; done
done
