mkdir -p gpurun_out
./tools/micro/shellsim > gpurun_out/micro.log 2>&1
cat gpurun_out/micro.log
