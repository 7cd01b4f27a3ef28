mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_shells" -s 1 -c 1 -o gpurun_out/prof_shells $CMD > gpurun_out/ncu_shells.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_shells.log
