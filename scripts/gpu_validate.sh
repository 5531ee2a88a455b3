# round-1 re-entry validation: GPU tests, smoke, bench, one ncu --set full of k_schur
set -x
TAG=${TAG:-val}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-ipm"
$CMD > gpurun_out/${TAG}_bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schur -s 1 -c 1 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log; tail -1 gpurun_out/${TAG}_bench.log
