mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt"
$B > gpurun_out/k1_plain.json 2> gpurun_out/k1_plain.err && \
ncu --set full --import-source on --clock-control none -k regex:k1_bulk --launch-skip 204 --launch-count 1 -o gpurun_out/ncu_k1_m_v4 $B > gpurun_out/ncu_k1b.log 2>&1
