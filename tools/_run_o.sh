for rep in 1 2 3; do for v in nopf k1pf; do
  FSQR_LIB=build_var/$v/libfsqr.so python bench.py --no-e2e --no-cpu --no-kkt --min-window 0.5 > gpurun_out/o_m_${v}_$rep.json 2>/dev/null
done; done
B="python bench.py --steps 3 --warmup 3 --burn-in 200 --no-e2e --no-cpu --no-kkt --min-window 0"
FSQR_LIB=build_var/k1pf/libfsqr.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k2_tc2|k1_tcp" -c 500 --csv --log-file gpurun_out/o_launches_k1pf.csv $B > gpurun_out/o_ncu.log 2>&1
