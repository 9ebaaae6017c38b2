set -x
python -m pytest tests -m "gpu and not fullsize" -q -x > gpurun_out/a_pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1
python bench.py --no-e2e --no-cpu --no-kkt > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
python tools/k1_timing.py > gpurun_out/a_k1t.txt 2>&1
python tools/bench_configs.py --configs c2,c5 --pack2 --no-kkt --steps 30 --burn-in 200 > gpurun_out/a_cfg.jsonl 2> gpurun_out/a_cfg.err
