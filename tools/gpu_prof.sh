# Profiles of the current build (GPU box): ncu --set full of one step_ring
# launch (cfg4 and forced cfg4) and the launch list of a short bench run.
#   gpurun -- 'bash tools/gpu_prof.sh <tag>'
tag=${1:-rNN}
cp paper_1208_2428_b200/lib/libfhpg.so paper_1208_2428_b200/lib/ab/$tag.so
bash tools/ncu_ab.sh $tag
timeout 600 ncu --set full --import-source on --clock-control none -k regex:step_ring -s 2 -c 1 \
  -o gpurun_out/ncu_${tag}_forced -f python tools/profile_step.py 4 16384 16384 fhp3 0.01 > gpurun_out/ncu_${tag}_forced.log 2>&1; echo forced=$?
ncu -i gpurun_out/ncu_${tag}_forced.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_forced_raw.csv 2>/dev/null
ncu -i gpurun_out/ncu_${tag}_forced.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${tag}_forced_sass.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches_$tag.log 2>&1; echo launches=$?
