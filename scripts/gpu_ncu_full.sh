# One `ncu --set full --import-source on` capture of k_schur on config ${CFG:-4} (the second launch),
# after the same command has run clean without ncu.  Output: gpurun_out/${TAG}_prof.ncu-rep
TAG=${TAG:-full}
CFG=${CFG:-4}
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${TAG}_plain.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_schur -s 1 -c 1 -f -o gpurun_out/${TAG}_prof $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
ls -la gpurun_out/${TAG}_prof.ncu-rep
