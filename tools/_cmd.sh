o=gpurun_out/r01r; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
bash tools/envsweep.sh "c2 c2d c5ag c3 c4 c5rs c1" "GC3_L2HINT=1;GC3_L2HINT=0" > $o/env.txt 2>&1
bash tools/gpu_ncu.sh r01r "c5ag"
