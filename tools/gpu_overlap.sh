run() { timeout -s KILL 600 env $1 python bench.py --no-cpu --no-e2e --no-extras --steps 10 $2 > gpurun_out/ov.json 2> gpurun_out/ov.err; python -c "
import json; d=json.loads(open('gpurun_out/ov.json').read().strip().splitlines()[-1]); print('$1 $2', 'C2', round(d['ms_per_step'],4), 'C5 us/frame', round(d['c5']['ms_per_frame_per_gpu']*1e3,2))" || tail -3 gpurun_out/ov.err; }
run X=1 "--chunk 64"
run X=1 "--chunk 32 --streams 2"
run GF_SHELL_BPS=1 "--chunk 32 --streams 2"
run GF_SHELL_BPS=1 "--chunk 16 --streams 2"
run GF_SHELL_BPS=1 "--chunk 32 --streams 1"
