D=paper_1611_05319_b200
for v in nosolo gsA gsB; do
  echo "== $v"
  GF_B200_LIB=$PWD/$D/libgf_b200_$v.so timeout -s KILL 600 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench_$v.json 2> gpurun_out/bench_$v.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_$v.json').read().strip().splitlines()[-1]); print('C2 ms', round(d['ms_per_step'],4), 'C5 ms/frame', round(d['c5']['ms_per_frame_per_gpu'],4))"
done
for v in gsA gsB; do
  echo "== trace $v"
  GF_B200_LIB=$PWD/$D/libgf_b200_$v.so timeout -s KILL 600 python tools/exp_deadlock.py --trace 2>&1 | cut -c1-300
done
