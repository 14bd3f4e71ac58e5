o=gpurun_out/r01ab; mkdir -p $o
bash tools/envsweep.sh "c2 c2d c5ag c5rs c3 c4" "GC3_L2HINT=3;GC3_L2HINT=1" > $o/env.txt 2>&1
