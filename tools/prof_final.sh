# round-1 evidence: full-size parity, default bench line (M, u8 input repacked to 2 bits), launch
# list of the profiled window, ncu --set full of the K2 and K1 kernels
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m fullsize -q > gpurun_out/pytest_full_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt"
$B > gpurun_out/pf_plain.json 2> gpurun_out/pf_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_tc|k1_|k_finalize" -c 2000 --csv --log-file gpurun_out/launches_m_final.csv $B > gpurun_out/ncu_lf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_tc2_kernel --launch-skip 206 --launch-count 1 -o gpurun_out/ncu_k2_m_final $B > gpurun_out/ncu_k2f.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_tcp_kernel --launch-skip 207 --launch-count 1 -o gpurun_out/ncu_k1_m_final $B > gpurun_out/ncu_k1f.log 2>&1
