timeout -s KILL 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
timeout -s KILL 600 python tools/exp_deadlock.py --reps 2 2>&1 | tee gpurun_out/exp_dl.json
GF_NO_SOLO=1 timeout -s KILL 600 python tools/exp_deadlock.py --reps 1 2>&1 | head -3
timeout -s KILL 900 python bench.py --no-cpu --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]); print('C2 ms', d['ms_per_step'], 'C5 ms/frame', d['c5']['ms_per_frame_per_gpu'], d['c5']['roofline']['frac'])"; tail -5 gpurun_out/bench.err
