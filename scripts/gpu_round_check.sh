# round-end style check: GPU tests, smoke, default bench, reference arm, cfg 5 bench
set -x
TAG=${TAG:-rc}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg5.log 2>&1
tail -2 gpurun_out/${TAG}_tests.log; tail -1 gpurun_out/${TAG}_smoke.log
