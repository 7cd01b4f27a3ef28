mkdir -p gpurun_out
CMD="python bench.py --frames 64 --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/plain_b.log 2>&1; echo "plain rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_shells|k_prep" -s 6 -c 2 -o gpurun_out/prof_batch $CMD > gpurun_out/ncu_b.log 2>&1; echo "full rc=$?"
