# per-variant timing + DRAM / L2 traffic of k_schur (single-pass ncu metrics, bytes only)
set -x
python tools/schur_exp.py run 4 > gpurun_out/${TAG}_exp.log 2>&1
for v in $(echo "$EXP_VARIANTS" | tr ';' '\n' | cut -d: -f1); do
  POLYA_LIB=build/exp/libpolya_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,gpu__time_duration.sum -k regex:k_schur -s 1 -c 1 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-ipm > gpurun_out/${TAG}_dram_$v.log 2>&1
done
