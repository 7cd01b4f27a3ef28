for c in 32 64 128 256; do
timeout -s KILL 600 python bench.py --no-cpu --no-e2e --steps 10 --chunk $c > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_c$c.json').read().strip().splitlines()[-1]); print('chunk $c C5 us/frame', round(d['c5']['ms_per_frame_per_gpu']*1e3,2), 'frac', round(d['c5']['roofline']['frac'],3))"
done
