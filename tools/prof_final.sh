# round-1 evidence: full-size parity, default bench line, launch list of the timed window, ncu of K2/K1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m fullsize -q > gpurun_out/pytest_full_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_full_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt"
$B > gpurun_out/pf_plain.json 2> gpurun_out/pf_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_tc|k1_bulk|k_finalize" --launch-skip 609 -c 9 --csv --log-file gpurun_out/launches_m_final.csv $B > gpurun_out/ncu_lf.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k2_tc_kernel --launch-skip 204 --launch-count 1 -o gpurun_out/ncu_k2_m_final $B > gpurun_out/ncu_k2f.log 2>&1
