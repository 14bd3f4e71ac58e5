o=gpurun_out/r01ap; mkdir -p $o
bash tools/envsweep.sh "c1 c4" "GC3_TILE_BYTES=2048;GC3_TILE_BYTES=4096;GC3_TILE_BYTES=8192;GC3_TILE_BYTES=16384" "--proto ll" > $o/env.txt 2>&1
bash tools/envsweep.sh "c1" "GC3_UNIT_WARPS=8;GC3_UNIT_WARPS=16;GC3_UNIT_WARPS=2" "--proto ll" >> $o/env.txt 2>&1
for t in 2048 4096; do GC3_TILE_BYTES=$t timeout 300 python bench.py --config c4 --sweep --sweep-min 1024 --sweep-max 8388608 --sweep-protos ll --steps 20 > $o/sweep_t$t.jsonl 2>&1; done
