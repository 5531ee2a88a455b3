set -x
mkdir -p gpurun_out
ITERS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_block_lmin -s 0 -c 1 -o gpurun_out/lmin_prof python scripts/ipm_step_run.py 4 > gpurun_out/lmin_prof.log 2>&1

ls -la gpurun_out
