# round-2 ncu evidence at M (u8 input repacked to 2 bits): launch list of the hot-path kernels and
# one --set full capture each of K1 (forward product + fused finalize) and K2
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt --min-window 0"
$B > gpurun_out/pf_plain.json 2> gpurun_out/pf_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_tc|k1_|k_finalize" -c 2000 --csv --log-file gpurun_out/r02_launches_m.csv $B > gpurun_out/ncu_lf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_tcp_kernel --launch-skip 205 --launch-count 1 -o gpurun_out/r02_ncu_k1_m $B > gpurun_out/ncu_k1.log 2>&1
