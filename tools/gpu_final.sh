# Final refresh (GPU box): smoke, full GPU suite, bench + reference arm, configs,
# profiles (ncu full + forced + launch list), multi-strip overheads, sanitizer.
#   gpurun -- 'bash tools/gpu_final.sh <tag>'
tag=${1:-rNN}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$tag.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu_$tag.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu_$tag.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; echo ref=$?
timeout 300 python tools/bench_configs.py > gpurun_out/configs_$tag.json 2>&1; echo configs=$?
bash tools/gpu_prof.sh $tag
timeout 600 python tools/multi_overhead.py 100 2 4 > gpurun_out/multi_overhead_$tag.json 2>&1; echo multi=$?
timeout 600 python tools/strip_overhead.py 100 > gpurun_out/strip_overhead_$tag.json 2>&1; echo strip=$?
# compute-sanitizer is closed on the GPU pool since r02w (profiles/sanitizer_r02v.txt is the last pass):
# bash tools/gpu_sanitize.sh $tag
