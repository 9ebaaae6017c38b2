mkdir -p gpurun_out
python bench.py --no-cpu --no-e2e --no-kkt > gpurun_out/bench_graph.json 2> gpurun_out/bench_graph.err
C="python bench.py --config c4 --steps 2 --warmup 3 --burn-in 30 --no-e2e --no-cpu --no-kkt"
$C > gpurun_out/p_c4b.json 2> gpurun_out/p_c4b.err && \
ncu --set full --import-source on --clock-control none -k regex:k2_tc2 --launch-skip 34 --launch-count 1 -o gpurun_out/ncu_tc2_v3 $C > gpurun_out/ncu_tc2c.log 2>&1
F="python tools/bench_configs.py --configs c5 --no-kkt --steps 3 --burn-in 20"
$F > gpurun_out/p_c5.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2_tc_kernel --launch-skip 30 --launch-count 1 -o gpurun_out/ncu_k2_c5 $F > gpurun_out/ncu_c5.log 2>&1
