# build -> parity tests -> timing variants (tools/schur_exp.py) on the GPU box
set -x
TAG=${TAG:-iter}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
tail -3 gpurun_out/${TAG}_tests.log
python tools/schur_exp.py run ${CFG:-4} > gpurun_out/${TAG}_exp.log 2>&1
cat gpurun_out/${TAG}_exp.log
