o=gpurun_out/r01ao; mkdir -p $o
timeout 900 python -m pytest tests -m gpu -q > $o/pytest_gpu.log 2>&1; echo "rc=$?" >> $o/pytest_gpu.log
for c in c1 c2 c3 c4 c5rs c5ag c2d; do timeout 120 python bench.py --config $c --quick --steps 20 >> $o/quick.jsonl 2>&1; done
