timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "eta or colstats" > gpurun_out/j_pytest.log 2>&1
python tools/setup_profile.py m 2 > gpurun_out/j_setup_m.json 2> gpurun_out/j_setup_m.err
python tools/setup_profile.py c4 2 > gpurun_out/j_setup_c4.json 2> gpurun_out/j_setup_c4.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/j_setup_launches.csv python tools/setup_profile.py m 1 > gpurun_out/j_setup_ncu.log 2>&1
