#!/bin/bash
# Tuning sweep (runs on the GPU box): kernel build variants x unit sizes x configs.
# usage: tools/tune.sh "T512U4B2 T512U8B1" "c2 c3" "4 8"
variants=${1:-"T512U8B1"}
configs=${2:-"c2"}
uws=${3:-"4"}
for v in $variants; do
  t=$(echo $v | sed -E 's/T([0-9]+)U([0-9]+)B([0-9]+)/\1/'); u=$(echo $v | sed -E 's/T([0-9]+)U([0-9]+)B([0-9]+)/\2/'); b=$(echo $v | sed -E 's/T([0-9]+)U([0-9]+)B([0-9]+)/\3/')
  GC3_BUILD_TAG=_$v GC3_LIB_OUT=/tmp/libgc3_$v.so GC3_NVCC_DEFS="-DGC3_THREADS=$t -DGC3_UNROLL=$u -DGC3_MINBLOCKS=$b" \
    python -m paper_2201_11840_b200.build > /tmp/build_$v.log 2>&1 || { echo "build $v failed"; tail -5 /tmp/build_$v.log; continue; }
  for uw in $uws; do
    for c in $configs; do
      r=$(GC3_LIB_PATH=/tmp/libgc3_$v.so GC3_UNIT_WARPS=$uw timeout 120 python bench.py --config $c --quick --steps 10 ${EXTRA} 2>&1 | tail -1)
      echo "$v uw=$uw $r"
    done
  done
done
