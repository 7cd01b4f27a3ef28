mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_copy|k_prep" -s 2 -c 2 -o gpurun_out/prof_prep $CMD > gpurun_out/ncu_prep.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_prep.log
