# K4 timing variants (tools/schur_exp.py): parity of each variant on configs 1-3, then bench at configs 4 and 3
set -x
mkdir -p gpurun_out
export EXP_VARIANTS=${EXP_VARIANTS:-"base:"}   # e.g. "base:;noepi:SCHUR_EXP=1" (the -D knobs csrc/schur.cu defines)
TAG=${TAG:-exp}
for v in $(echo "$EXP_VARIANTS" | tr ';' '\n' | cut -d: -f1 | grep -v '^base$'); do
  POLYA_LIB=build/exp/libpolya_$v.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "schur_full_parity or pair_tiles or rank_sharding or schur_config3 or size_boundary" > gpurun_out/${TAG}_parity_$v.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_parity_$v.log
done
for c in ${CFGS:-4 3}; do timeout 900 python tools/schur_exp.py run $c > gpurun_out/${TAG}_cfg$c.log 2>&1; done
tail -n 2 gpurun_out/${TAG}_parity_*.log; cat gpurun_out/${TAG}_cfg*.log
