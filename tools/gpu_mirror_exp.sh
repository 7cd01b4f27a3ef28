python tools/exp_mirror.py > gpurun_out/e2e_delta2.log 2>&1; echo rc=$?; cat gpurun_out/e2e_delta2.log
