# Smoke, the full GPU suite, the bench line and the BASELINE config shapes (GPU box):
#   gpurun -- 'bash tools/gpu_check.sh <tag>'
tag=${1:-r02k}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?; tail -1 gpurun_out/bench_$tag.json | cut -c1-1200; tail -3 gpurun_out/bench_$tag.err
timeout 300 python tools/bench_configs.py > gpurun_out/configs_$tag.json 2>&1; echo configs=$?; cut -c1-220 gpurun_out/configs_$tag.json
