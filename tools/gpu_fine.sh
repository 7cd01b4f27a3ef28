mkdir -p gpurun_out
: > gpurun_out/fine.log
for v in fine; do
  echo "== $v" >> gpurun_out/fine.log
  GF_B200_LIB=paper_1611_05319_b200/libgf_b200_$v.so timeout -s KILL 300 python tools/exp_fine.py C2 >> gpurun_out/fine.log 2>&1
done
cat gpurun_out/fine.log
./tools/micro/lat >> gpurun_out/fine.log 2>&1; tail -12 gpurun_out/fine.log
