for rep in 1 2; do
  for v in s0 cur; do
    FSQR_LIB=build_var/$v/libfsqr.so python tools/bench_configs.py --configs c4 --no-kkt --steps 30 --burn-in 200 > gpurun_out/m_c4_${v}_$rep.jsonl 2>/dev/null
  done
  for pr in 2 1 0; do
    FSQR_L2PROMO=$pr python bench.py --no-e2e --no-cpu --no-kkt --min-window 0.5 > gpurun_out/m_m_promo${pr}_$rep.json 2>/dev/null
  done
done
