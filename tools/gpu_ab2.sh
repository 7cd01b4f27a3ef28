mkdir -p gpurun_out
GF_B200_LIB=$PWD/paper_1611_05319_b200/libgf_b200_f32rot.so timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_f32rot.log 2>&1; echo "variant pytest rc=$?"; tail -3 gpurun_out/pytest_f32rot.log
LIBS="libgf_b200.so libgf_b200_f32rot.so libgf_b200.so libgf_b200_f32rot.so" bash tools/gpu_ab.sh 2>&1 | grep -E "rc=|ms/frame"
for cfg in C3 C4; do for lib in libgf_b200.so libgf_b200_f32rot.so; do GF_B200_LIB=$PWD/paper_1611_05319_b200/$lib timeout 300 python bench.py --config $cfg --steps 50 --no-cpu --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $lib', round(d['ms_per_step'],4))"; done; done
