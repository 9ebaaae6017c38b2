mkdir -p gpurun_out
python tools/k1_exp2.py save m 1 > gpurun_out/k1tcp_save.log 2>&1
python tools/k1_exp2.py time m 1 tcp > gpurun_out/k1tcp_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k1_tcp --launch-skip 6 --launch-count 1 -o gpurun_out/ncu_k1tcp_m python tools/k1_exp2.py time m 1 tcp > gpurun_out/ncu_k1tcp.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k1_bulk --launch-skip 6 --launch-count 1 -o gpurun_out/ncu_k1bulk_m python tools/k1_exp2.py time m 1 bulk > gpurun_out/ncu_k1bulk.log 2>&1
tail -2 gpurun_out/k1tcp_plain.log
