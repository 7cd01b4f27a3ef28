for lib in libgf_b200_lg4r4.so libgf_b200_lg4r5.so; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout 600 python -m pytest tests/test_gpu_configs.py -m gpu -x -q -k "config_parity or large_ball" 2>&1 | tail -1 | sed "s/^/$lib parity: /"
done
for rep in 1 2; do for cfg in C3 C4; do for lib in libgf_b200.so libgf_b200_lg4r4.so libgf_b200_lg4r5.so; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout 300 python bench.py --config $cfg --steps 50 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $lib', round(d['ms_per_step'],4))"
done; done; done
