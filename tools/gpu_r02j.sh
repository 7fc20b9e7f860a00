# round-2 re-entry check: smoke, full GPU suite, bench line, configs
tag=r02j
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
tail -25 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?; tail -1 gpurun_out/bench_$tag.json | cut -c1-1500; tail -3 gpurun_out/bench_$tag.err
timeout 300 python tools/bench_configs.py > gpurun_out/configs_$tag.json 2>&1; echo configs=$?; head -40 gpurun_out/configs_$tag.json
