timeout -s KILL 400 python -m pytest tests/test_gpu_deadlock.py tests/test_gpu_parity.py tests/test_gpu_coherence.py -q -x --timeout=120 2>&1 | tail -2
timeout -s KILL 300 python tools/exp_deadlock.py --reps 2 2>&1
timeout -s KILL 900 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('C2 ms', d['ms_per_step'], 'C5 ms/frame', d['c5']['ms_per_frame_per_gpu'])"
