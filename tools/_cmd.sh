o=gpurun_out/r01e; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
bash tools/ab.sh "old:-DGC3_TAIL_UNROLL=1 -DGC3_MOVE_NOINLINE=0;t4i:-DGC3_TAIL_UNROLL=4 -DGC3_MOVE_NOINLINE=0;t4n:-DGC3_TAIL_UNROLL=4 -DGC3_MOVE_NOINLINE=1;t2n:-DGC3_TAIL_UNROLL=2 -DGC3_MOVE_NOINLINE=1" "c1 c2 c3 c4 c5rs" > $o/ab.txt 2>&1
bash tools/ab.sh "t4nll:-DGC3_TAIL_UNROLL=4 -DGC3_MOVE_NOINLINE=1" "c1 c4" "--proto ll" >> $o/ab.txt 2>&1
bash tools/ab.sh "oldll:-DGC3_TAIL_UNROLL=1 -DGC3_MOVE_NOINLINE=0" "c1 c4" "--proto ll" >> $o/ab.txt 2>&1
