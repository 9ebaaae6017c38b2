mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:k2_tc2 --launch-skip 2 --launch-count 1 -o gpurun_out/ncu_c5_pack2_k2 \
  python tools/bench_configs.py --configs c5 --pack2 --no-kkt --steps 5 --burn-in 200 > gpurun_out/ncu_c5p.log 2>&1
