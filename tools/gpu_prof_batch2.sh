python tools/prof_batch.py 32
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/prof_batch.py 32 > gpurun_out/batch_launches.csv 2> gpurun_out/batch_launches.err; tail -12 gpurun_out/batch_launches.csv
timeout -s KILL 900 ncu --set full --import-source on --clock-control none -k regex:k_shells -s 2 -c 1 -o gpurun_out/batch_shells python tools/prof_batch.py 32 > /dev/null 2>&1; echo "ncu rc=$?"
