# A/B/.. of library variants: C2 ms/frame and C5 us/frame, interleaved twice.
# usage: bash tools/gpu_ab_multi.sh base new pb5 ...   (libgf_b200_<v>.so; "new" = libgf_b200.so)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    lib=$PWD/paper_1611_05319_b200/libgf_b200_$v.so; [ "$v" = new ] && lib=$PWD/paper_1611_05319_b200/libgf_b200.so
    GF_B200_LIB=$lib timeout -s KILL 600 python bench.py --no-cpu --no-e2e --no-extras --steps 30 > gpurun_out/abm_$v.json 2> gpurun_out/abm_$v.err
    python -c "
import json; d=json.loads(open('gpurun_out/abm_$v.json').read().strip().splitlines()[-1])
print('$v C2 ms', round(d['ms_per_step'],4), 'C5 us/frame', round(d['c5']['ms_per_frame_per_gpu']*1e3,2))"
  done
done
