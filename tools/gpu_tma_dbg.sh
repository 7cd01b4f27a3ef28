export CUDA_LAUNCH_BLOCKING=1
for d in f32 f64; do timeout 60 python tools/tma_dbg.py $d 2>&1 | tail -1; done
