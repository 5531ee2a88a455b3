# IPM kernels: parity tests of the step / solve / general forms, then plain + ncu launch list of 2-3 IPM steps (cfg 4)
set -x
TAG=${TAG:-ipm}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ipm.py tests/test_gpu_solve.py tests/test_gpu_general.py tests/test_gpu_dist.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
tail -3 gpurun_out/${TAG}_tests.log
ITERS=3 python scripts/ipm_step_run.py ${CFG:-4} > gpurun_out/${TAG}_plain.log 2>&1 && \
ITERS=2 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/ipm_step_run.py ${CFG:-4} > gpurun_out/${TAG}_ncu.log 2>&1
cat gpurun_out/${TAG}_plain.log
python scripts/launch_summary.py gpurun_out/${TAG}_launches.csv 2>&1 | head -30
