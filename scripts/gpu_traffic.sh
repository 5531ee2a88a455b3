# DRAM / L2 traffic of k_schur per variant (EXP_VARIANTS as in tools/schur_exp.py; build them first)
set -x
for v in $(echo "$EXP_VARIANTS" | tr ';' '\n' | cut -d: -f1); do
  POLYA_LIB=build/exp/libpolya_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum -k regex:k_schur -s 1 -c 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/${TAG}_traffic_$v.log 2>&1
done
