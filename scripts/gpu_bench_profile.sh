set -x
python bench.py > gpurun_out/bench1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref1.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv $CMD > gpurun_out/ncu1.log 2>&1
$CMD > gpurun_out/bench_small2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_schur -s 1 -c 1 -o gpurun_out/prof_schur1 $CMD > gpurun_out/ncu2.log 2>&1
echo done
