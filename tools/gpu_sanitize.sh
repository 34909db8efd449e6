# compute-sanitizer on the 8-CTA (24^3) and 16-CTA (32^3, C3 path) clusters, 200 iterations; raw logs kept
S=/usr/local/cuda/bin/compute-sanitizer
for case in "32 200" "24 200"; do
  set -- $case
  for tool in racecheck synccheck memcheck; do
    timeout 1200 $S --tool $tool --print-limit 50 python tools/sanitize_cluster.py $1 $2 > gpurun_out/sanitize_${tool}_$1.log 2>&1
    echo "n=$1 $tool rc=$?: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard|iters' gpurun_out/sanitize_${tool}_$1.log | tr '\n' ' ')"
  done
done
