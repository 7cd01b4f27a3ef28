# Full bench line + reference arm + ncu launch list + full capture of both fill kernels.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.csv
timeout -s KILL 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"
timeout -s KILL 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
timeout -s KILL 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"k_shells|k_prep" -s 6 -c 2 -o gpurun_out/prof_${TAG:-final} $CMD > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -c 1500 gpurun_out/bench_full.log; echo; tail -c 700 gpurun_out/bench_ref.log
