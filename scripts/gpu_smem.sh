# shared-memory wavefronts / bank conflicts of k_schur per variant (single ncu pass)
for v in $(echo "$EXP_VARIANTS" | tr ';' '\n' | cut -d: -f1); do
  POLYA_LIB=build/exp/libpolya_$v.so timeout 600 ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,smsp__inst_executed_op_ldgsts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed.sum -k regex:k_schur -s 1 -c 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/${TAG}_smem_$v.log 2>&1
done
