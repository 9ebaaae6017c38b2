# run B: C5 K2 source-level ncu, setup breakdown, K1 ncu at M
mkdir -p gpurun_out
python tools/setup_profile.py m 2 > gpurun_out/b_setup_m.json 2> gpurun_out/b_setup_m.err
python tools/setup_profile.py c4 1 > gpurun_out/b_setup_c4.json 2> gpurun_out/b_setup_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/b_setup_launches.csv python tools/setup_profile.py m 1 > gpurun_out/b_setup_ncu.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_tc2 --launch-skip 2 --launch-count 1 -o gpurun_out/b_ncu_c5_k2 \
  python tools/bench_configs.py --configs c5 --pack2 --no-kkt --steps 5 --burn-in 200 > gpurun_out/b_ncu_c5.log 2>&1
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt --min-window 0"
ncu --set full --import-source on --clock-control none -k regex:k1_tcp_kernel --launch-skip 205 --launch-count 1 -o gpurun_out/b_ncu_k1_m $B > gpurun_out/b_ncu_k1.log 2>&1
python tools/k1_timing.py > gpurun_out/b_k1t.txt 2>&1
for v in nl nu nm na; do K1T=k1t_$v python tools/k1_timing.py > gpurun_out/b_k1t_$v.txt 2>&1; done
