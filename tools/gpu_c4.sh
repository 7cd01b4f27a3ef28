for lib in ${LIBS:-libgf_b200.so}; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout -s KILL 600 python bench.py --config C4 --steps 30 --no-cpu --no-e2e > gpurun_out/bench_C4_$lib.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_C4_$lib.log').read().strip().splitlines()[-1]); print('$lib', 'C4 ms/frame %.4f' % d['ms_per_step'])"
done
