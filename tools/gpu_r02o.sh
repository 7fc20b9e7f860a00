# round-2 refresh: bench line, configs, profiles (ncu full + forced + launches), multi-strip overhead
tag=${1:-r02o}
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; echo ref=$?
timeout 300 python tools/bench_configs.py > gpurun_out/configs_$tag.json 2>&1; echo configs=$?
bash tools/gpu_prof.sh $tag
timeout 600 python tools/multi_overhead.py 100 2 4 > gpurun_out/multi_overhead_$tag.json 2>&1; echo multi=$?; cat gpurun_out/multi_overhead_$tag.json
timeout 600 python tools/strip_overhead.py 100 > gpurun_out/strip_overhead_$tag.json 2>&1; echo strip=$?; tail -1 gpurun_out/strip_overhead_$tag.json
