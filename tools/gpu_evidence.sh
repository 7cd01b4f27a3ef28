# Full bench line + reference arm + ncu launch list + full capture of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.csv
timeout -s KILL 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_shells|k_prep|k_copy|k_finalize" -s 4 -c 4 -o gpurun_out/prof_final $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
