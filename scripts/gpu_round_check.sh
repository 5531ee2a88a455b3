# round-end style check: GPU tests, smoke, default bench, block-shard bench, reference arm, cfg 5 bench,
# launch list of the default bench command (ncu, after it ran clean)
set -x
TAG=${TAG:-rc}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
python bench.py > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
python bench.py --shard blocks --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_blocks.log 2>&1
python bench.py --shard blocks --combine p2p --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_p2p.log 2>&1
python bench.py --impl reference > gpurun_out/${TAG}_ref.log 2>&1
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg5.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
tail -3 gpurun_out/${TAG}_tests.log; tail -1 gpurun_out/${TAG}_smoke.log
for f in gpurun_out/${TAG}_bench.log gpurun_out/${TAG}_bench_blocks.log gpurun_out/${TAG}_bench_p2p.log gpurun_out/${TAG}_bench_cfg5.log gpurun_out/${TAG}_ref.log; do tail -1 $f | cut -c1-200; done
