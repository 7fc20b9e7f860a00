# compute-sanitizer over every step kernel (GPU box):
#   gpurun -- 'bash tools/gpu_sanitize.sh <tag>'  -> gpurun_out/sanitizer_<tag>.txt
tag=${1:-rNN}
out=gpurun_out/sanitizer_$tag.txt
: > $out
for tool in memcheck racecheck initcheck synccheck; do
  echo "== compute-sanitizer --tool $tool python tools/sanitize.py" >> $out
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py >> $out 2>&1
  echo "rc=$?" >> $out
done
grep -E "SUMMARY|rc=|^==" $out
