o=gpurun_out/r01am; mkdir -p $o
for n in 1 2 4; do GC3_E2E_STREAMS=$n timeout 300 python bench.py --no-cpu-baseline > $o/bench_s$n.json 2>&1; done
