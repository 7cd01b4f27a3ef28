set -x
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" ; grep -o -w -E "avx512f|avx512bw|avx512vl|avx512dq|avx2|fma" /proc/cpuinfo | sort | uniq -c
python -c "from oracle import guidefill_oracle as o; print('numpy exp flavour:', o.numpy_exp_flavour())"
timeout -s KILL 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -20 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
