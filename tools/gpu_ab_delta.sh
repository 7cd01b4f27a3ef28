# A/B of gf_output_delta (coalesced host writes, new) vs one store per channel (old lib).
for rep in 1 2; do
  for v in old new; do
    if [ $v = old ]; then L=paper_1611_05319_b200/libgf_b200_old.so; else L=paper_1611_05319_b200/libgf_b200.so; fi
    echo "== $v"; GF_B200_LIB=$L timeout 200 python tools/e2e_breakdown.py 2>&1 | grep -E "run_tracked|finish"
  done
done
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
