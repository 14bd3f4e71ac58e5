o=gpurun_out/r01af; mkdir -p $o
bash tools/ab.sh "llb1:-DGC3_LL_BATCH=1;llb2:-DGC3_LL_BATCH=2;llb4:-DGC3_LL_BATCH=4" "c1 c4" "--proto ll" > $o/ab.txt 2>&1
for L in 1 4; do GC3_LIB_PATH=/tmp/libgc3_llb$L.so timeout 300 python bench.py --config c4 --sweep --sweep-min 1024 --sweep-max 8388608 --sweep-protos ll --steps 20 > $o/sweep_b$L.jsonl 2>&1; done
