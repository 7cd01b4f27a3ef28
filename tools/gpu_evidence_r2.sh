# Round-2 evidence: full bench line, reference arm, GPU suite, ncu launch list + full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.csv
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/cpu_info.txt
timeout -s KILL 900 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c5 --no-extras"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prep|k_shells" --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_shells|k_prep" -s 6 -c 2 -o gpurun_out/prof_r2 $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -c 1200 gpurun_out/bench_full.log; echo; tail -c 600 gpurun_out/bench_ref.log
