mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt"
FSQR_K1=tc $B > gpurun_out/k1tc_plain.json 2> gpurun_out/k1tc_plain.err && \
FSQR_K1=tc ncu --set full --import-source on --clock-control none -k regex:k1_tc_kernel --launch-skip 204 --launch-count 1 -o gpurun_out/ncu_k1tc $B > gpurun_out/ncu_k1tc.log 2>&1
