mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/k3b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/k3b_tests.log
for c in 4 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/k3b_bench_cfg$c.log 2>&1; done
timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/k3b_bench_cfg5.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k3b_launches.csv $CMD > /dev/null 2>&1
tail -n 3 gpurun_out/k3b_tests.log
