# full bench lines (cfg 4 default and cfg 5) + reference arm, round-1 measurement script
set -x
python bench.py > gpurun_out/${TAG}_bench_cfg4.log 2>&1
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg5.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.log 2>&1
nvidia-smi --query-gpu=memory.used,memory.total --format=csv > gpurun_out/${TAG}_mem.txt
