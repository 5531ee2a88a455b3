# one build -> test -> bench -> profile iteration on the GPU box (round-1 working script)
set -x
TAG=${TAG:-iter}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
tail -3 gpurun_out/${TAG}_tests.log
CMD="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_bench.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_schur -s 1 -c 1 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_bench.log
