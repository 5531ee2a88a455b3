mkdir -p gpurun_out
for v in base w2; do
  export POLYA_LIB=build/exp/libpolya_$v.so
  timeout 300 python tools/k4_time.py 16 3 2 2 2 3 --parity
  timeout 300 python tools/k4_time.py 24 4 2 2 2 3 --parity
  timeout 300 python tools/k4_time.py 96 4 2 4 4 5
  timeout 300 python tools/k4_time.py 104 4 2 4 4 5
  timeout 300 python tools/k4_time.py 32 4 2 3 3 5
  timeout 600 python tools/k4_time.py 120 6 2 4 4 3
done 2>&1 | grep -v Warning
