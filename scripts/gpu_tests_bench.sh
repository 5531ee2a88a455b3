# full GPU test suite + default bench line
set -x
TAG=${TAG:-tb}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
