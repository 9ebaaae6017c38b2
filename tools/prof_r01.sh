mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu"
$B > gpurun_out/p_plain.json 2> gpurun_out/p_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 640 --csv --log-file gpurun_out/launches_r01_v3.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_tc_kernel --launch-skip 204 --launch-count 1 -o gpurun_out/ncu_k2_m_v3 $B > gpurun_out/ncu_k2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_bulk --launch-skip 204 --launch-count 1 -o gpurun_out/ncu_k1_m_v3 $B > gpurun_out/ncu_k1.log 2>&1
C="python bench.py --config c4 --steps 2 --warmup 3 --burn-in 30 --no-e2e --no-cpu"
$C > gpurun_out/p_c4.json 2> gpurun_out/p_c4.err && \
ncu --set full --import-source on --clock-control none -k regex:k2_tc2 --launch-skip 34 --launch-count 1 -o gpurun_out/ncu_tc2_v2 $C > gpurun_out/ncu_tc2b.log 2>&1
