# round-2 session-3 final evidence at M (u8 input repacked to 2 bits): default bench line, launch list of the
# profiled window, ncu --set full of K2 and K1, per-config table (stored and repacked), tuning protocol, whole GPU suite
mkdir -p gpurun_out
python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt --min-window 0"
$B > gpurun_out/f_pf_plain.json 2> gpurun_out/f_pf_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_tc|k1_|k_finalize" -c 2000 --csv --log-file gpurun_out/f_launches_m.csv $B > gpurun_out/f_ncu_lf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_tc2_kernel --launch-skip 206 --launch-count 1 -o gpurun_out/f_ncu_k2_m $B > gpurun_out/f_ncu_k2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_tcp_kernel --launch-skip 207 --launch-count 1 -o gpurun_out/f_ncu_k1_m $B > gpurun_out/f_ncu_k1.log 2>&1
python tools/bench_configs.py --configs c1,c2,c3,c4,c5,m > gpurun_out/f_configs_stored.jsonl 2> gpurun_out/f_configs_stored.err
python tools/bench_configs.py --configs c2,c3,c5,m --pack2 > gpurun_out/f_configs_pack2.jsonl 2> gpurun_out/f_configs_pack2.err
python tools/tune_protocol.py --configs c2,m > gpurun_out/f_tune.jsonl 2> gpurun_out/f_tune.err
python -m pytest tests -m gpu -q --durations=8 > gpurun_out/f_pytest_gpu.log 2>&1; tail -2 gpurun_out/f_pytest_gpu.log; python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; cat gpurun_out/f_bench.json | cut -c1-300
