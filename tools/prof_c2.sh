# C2 (n=2000, p=50k): per-kernel device times (launch list) of the timed window + memcheck on the smoke test
mkdir -p gpurun_out
B="python bench.py --config c2 --steps 20 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt"
$B > gpurun_out/c2_plain.json 2> gpurun_out/c2_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k2_tc|k1_bulk|k_finalize" --launch-skip 609 -c 60 --csv --log-file gpurun_out/launches_c2.csv $B > gpurun_out/ncu_c2.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck_smoke.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/memcheck_smoke.log
