for rep in 1 2; do for v in fence nocv cw8; do
  FSQR_LIB=build_var/$v/libfsqr.so python tools/bench_configs.py --configs c5 --pack2 --no-kkt --steps 30 --burn-in 200 > gpurun_out/l_c5_${v}_$rep.jsonl 2>/dev/null
done; done
FSQR_LIB=build_var/nocv/libfsqr.so python bench.py --no-e2e --no-cpu --no-kkt --min-window 0.5 > gpurun_out/l_m_nocv.json 2>/dev/null
FSQR_LIB=build_var/cw8/libfsqr.so timeout 900 python -m pytest tests/test_gpu_pack2.py tests/test_gpu_parity.py tests/test_gpu_path_edges.py tests/test_gpu_api.py -q -x > gpurun_out/l_pytest_cw8.log 2>&1
