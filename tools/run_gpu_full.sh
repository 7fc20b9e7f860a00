# Full GPU pass for the round: smoke, the GPU test suite, the bench line
# (with e2e and the reference CPU baseline), the launch list of a short
# bench run and one ncu --set full capture of the step kernel.
#   gpurun -- 'bash tools/run_gpu_full.sh <tag>'
tag=${1:-rNN}
set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -14 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench=$?; tail -1 gpurun_out/bench_$tag.json | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$tag.json 2>&1; echo ref=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$tag.log 2>&1; echo launches=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:step_ring -s 2 -c 1 -o gpurun_out/prof_$tag python tools/profile_step.py 4 > gpurun_out/ncu_$tag.log 2>&1; echo ncu=$?
