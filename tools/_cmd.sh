o=gpurun_out/r01w; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
bash tools/ab.sh "wqnoinl:-DGC3_WQ_NOINLINE=1;wqinl:-DGC3_WQ_NOINLINE=0" "c2 c3 c4 c5rs c5ag c1" > $o/ab.txt 2>&1
