mkdir -p gpurun_out
F="python tools/iter_rhs.py --config c5 --burn-in 20 --steps 3"
$F > gpurun_out/c5_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k2_tc_kernel --launch-skip 21 --launch-count 1 -o gpurun_out/ncu_k2_c5 $F > gpurun_out/ncu_c5.log 2>&1
