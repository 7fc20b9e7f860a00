# GPU test pass + bench line: gpurun -- 'bash tools/gpu_tests.sh <tag> [pytest -k expr]'
tag=${1:-rNN}
kexpr=${2:-}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_$tag.log
if [ -n "$kexpr" ]; then
  timeout 2400 python -m pytest tests -m gpu -q --durations=12 -k "$kexpr" > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
else
  timeout 2400 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?
fi
tail -25 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?; tail -1 gpurun_out/bench_$tag.json | cut -c1-1500; tail -3 gpurun_out/bench_$tag.err
