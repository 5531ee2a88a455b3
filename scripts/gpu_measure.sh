# measurement bundle: default bench line, block-shard bench line, cfg 5 line, launch list, ncu --set full of k_schur
set -x
TAG=${TAG:-m}
python bench.py > gpurun_out/${TAG}_bench_cfg4.log 2>&1
python bench.py --shard blocks --steps 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_blocks.log 2>&1
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg5.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-ipm"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schur -s 1 -c 1 -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
for f in gpurun_out/${TAG}_bench_*.log; do tail -1 $f | cut -c1-200; done
