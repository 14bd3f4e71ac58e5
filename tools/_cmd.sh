mkdir -p gpurun_out/r01c
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01c/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r01c/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r01c/bench.json 2> gpurun_out/r01c/bench.err
bash tools/gpu_ncu.sh r01c "c1 c3 c4 c5rs"
