# Coherence-transport evidence: per-phase trace, timing, 1080p oracle parity, ncu capture.
mkdir -p gpurun_out
GF_CT_TRACE=1 timeout -s KILL 300 python tools/prof_coherence_loop.py --ncu > /dev/null 2> gpurun_out/ct_trace.txt
timeout -s KILL 300 python tools/prof_coherence_loop.py > gpurun_out/ct_time.json 2>&1
timeout -s KILL 600 python tools/exp_coherence.py > gpurun_out/ct_exp.json 2> gpurun_out/ct_exp.err; echo "exp rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:k_ct_loop -c 1 -o gpurun_out/prof_ctloop_final python tools/prof_coherence_loop.py --ncu > gpurun_out/ncu_ctloop.log 2>&1; echo "ncu rc=$?"
