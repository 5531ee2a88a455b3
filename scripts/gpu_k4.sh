# K4 measurement bundle (one gpurun call): schur parity tests, bench lines for configs 4 / 3 / 5 (assembly
# only), and an ncu pass of selected k_schur counters (time, DRAM, L2 reads, shared-memory wavefronts and
# bank conflicts by op, DMMA pipe) on config 4.  TAG names the outputs under gpurun_out/.
set -x
TAG=${TAG:-k4}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "schur or setup" > gpurun_out/${TAG}_tests.log 2>&1
tail -2 gpurun_out/${TAG}_tests.log
for C in 4 3; do
  python bench.py --config $C --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/${TAG}_bench_cfg$C.json 2> gpurun_out/${TAG}_bench_cfg$C.err
done
[ "${CFG5:-1}" = 1 ] && python bench.py --config 5 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ldgsts.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm"
timeout 900 ncu --metrics $M --clock-control none -k regex:k_schur -s 1 -c 1 --csv $CMD > gpurun_out/${TAG}_ncu_k4.csv 2> gpurun_out/${TAG}_ncu_k4.err
for f in gpurun_out/${TAG}_bench_cfg*.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['tflops_schur_assembly_only'],3), round(d['roofline']['frac'],4), d['breakdown_ms'])"; done
grep -E "k_schur" gpurun_out/${TAG}_ncu_k4.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}' | head -20
