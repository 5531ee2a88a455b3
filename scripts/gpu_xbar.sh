# per-variant timing + L2->SM traffic of k_schur (single-metric ncu pass, cold cache: bytes only)
set -x
python tools/schur_exp.py run 4 > gpurun_out/${TAG}_exp.log 2>&1
for v in $(echo "$EXP_VARIANTS" | tr ';' '\n' | cut -d: -f1); do
  POLYA_LIB=build/exp/libpolya_$v.so timeout 600 ncu --metrics l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,gpu__time_duration.sum -k regex:k_schur -s 1 -c 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/${TAG}_xbar_$v.log 2>&1
done
