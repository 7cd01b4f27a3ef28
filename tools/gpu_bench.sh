set -x
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/pytest_configs.log 2>&1; echo "configs rc=$?"; tail -15 gpurun_out/pytest_configs.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -5 gpurun_out/bench.log
timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --untracked --no-e2e --no-cpu > gpurun_out/bench_untracked.log 2>&1; echo "bench untracked rc=$?"; tail -3 gpurun_out/bench_untracked.log
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -3 gpurun_out/bench_ref.log
