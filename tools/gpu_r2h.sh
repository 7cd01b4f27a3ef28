timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_deadlock.py -q -x --timeout=300 2>&1 | tail -2
timeout -s KILL 900 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/bench.json 2> gpurun_out/bench.err; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); c=d['config']; print('C2 ms', round(d['ms_per_step'],4), 'C5 us/frame', round(d['c5']['ms_per_frame_per_gpu']*1e3,2), c['timeline'], [round(r['fill_us'],2) for r in c['shell_trace']])"
