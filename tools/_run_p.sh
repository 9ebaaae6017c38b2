FSQR_LIB=build_var/dec/libfsqr.so timeout 900 python -m pytest tests/test_gpu_pack2.py tests/test_gpu_parity.py -q -x > gpurun_out/p_pytest_dec.log 2>&1
for rep in 1 2; do for v in nopf dec; do
  FSQR_LIB=build_var/$v/libfsqr.so python tools/bench_configs.py --configs c5 --pack2 --no-kkt --steps 30 --burn-in 200 > gpurun_out/p_c5_${v}_$rep.jsonl 2>/dev/null
  FSQR_LIB=build_var/$v/libfsqr.so python bench.py --no-e2e --no-cpu --no-kkt --min-window 0.5 > gpurun_out/p_m_${v}_$rep.json 2>/dev/null
  FSQR_LIB=build_var/$v/libfsqr.so python tools/bench_configs.py --configs c4 --no-kkt --steps 30 --burn-in 200 > gpurun_out/p_c4_${v}_$rep.jsonl 2>/dev/null
done; done
