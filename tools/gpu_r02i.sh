timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 900 python -m pytest tests/test_resident_gpu.py tests/test_parity_gpu.py tests/test_planes_gpu.py -q -x 2>&1 | tail -5
timeout 300 python tools/bench_configs.py > gpurun_out/configs_r02i.json 2>&1; echo configs=$?; cat gpurun_out/configs_r02i.json | head -30
