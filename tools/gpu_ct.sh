# Coherence-loop iteration: per-phase trace, timing, coherence + parity tests.
mkdir -p gpurun_out
GF_CT_TRACE=1 timeout -s KILL 300 python tools/prof_coherence_loop.py --ncu > /dev/null 2> gpurun_out/ct_trace.txt
timeout -s KILL 300 python tools/prof_coherence_loop.py > gpurun_out/ct_time.json 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_coherence.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/ct_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/ct_tests.log
python -c "import json; d=json.load(open('gpurun_out/ct_time.json')); print('kernel', d['kernel_ms'], 'api', d['api_ms'])"
