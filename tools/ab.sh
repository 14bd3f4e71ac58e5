#!/bin/bash
# A/B of kernel build variants (runs on the GPU box): tools/ab.sh "NAME:DEFS;NAME:DEFS" "c1 c2 c3 c4" [extra bench args]
IFS=';' read -ra variants <<< "$1"
configs=${2:-"c1 c2 c3 c4"}
extra=${3:-}
for v in "${variants[@]}"; do
  name=${v%%:*}; defs=${v#*:}
  GC3_BUILD_TAG=_$name GC3_LIB_OUT=/tmp/libgc3_$name.so GC3_NVCC_DEFS="$defs" python -m paper_2201_11840_b200.build > /tmp/build_$name.log 2>&1 \
    || { echo "build $name failed"; tail -5 /tmp/build_$name.log; continue; }
  for c in $configs; do
    r=$(GC3_LIB_PATH=/tmp/libgc3_$name.so timeout 120 python bench.py --config $c --quick --steps 20 $extra 2>&1 | tail -1)
    echo "$name $c $r"
  done
done
