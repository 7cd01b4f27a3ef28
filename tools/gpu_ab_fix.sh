# A/B of a kernel change against the previous library (C2 / C5 / deadlock regime), then
# the parity tests and the random sweep.
mkdir -p gpurun_out
for v in b200_base b200 b200_base b200; do
  GF_B200_LIB=$PWD/paper_1611_05319_b200/libgf_$v.so timeout -s KILL 900 python bench.py --no-cpu --no-e2e --steps 30 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); dl=d['deadlock_regime']
print('$v C2 ms', round(d['ms_per_step'],4), 'C5 us/frame', round(d['c5']['ms_per_frame_per_gpu']*1e3,2), 'dl25', round(dl['halfplane_25deg_mu50']['us_per_shell'],2), 'dl10', round(dl['halfplane_10deg_mu50']['us_per_shell'],2))"
done
timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_deadlock.py tests/test_gpu_sweep.py -q -x -p no:cacheprovider > gpurun_out/fix_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/fix_tests.log
timeout -s KILL 900 python tools/sweep_fill.py 120 99 2>&1 | grep -v Warn | grep -v "conf =" | tail -3
