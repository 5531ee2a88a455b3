set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ll_build.log 2>&1
ITERS=3 python scripts/ipm_step_run.py 4 > gpurun_out/ll_ipm_plain.log 2>&1 && \
ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_ipm_launches.csv python scripts/ipm_step_run.py 4 > gpurun_out/ll_ncu.log 2>&1
cat gpurun_out/ll_ipm_plain.log
python scripts/launch_summary.py gpurun_out/ll_ipm_launches.csv 2>&1 | head -40
