# compute-sanitizer on the final kernel: 16-CTA hardware cluster (C3) and virtual clusters (FRB_VIRTUAL_ONLY), 200 iterations
S=/usr/local/cuda/bin/compute-sanitizer
for tool in racecheck synccheck memcheck; do
  timeout 1500 $S --tool $tool --print-limit 50 python tools/sanitize_cluster.py 32 200 --check > gpurun_out/sanitize2_${tool}_32.log 2>&1
  echo "hw n=32 $tool rc=$?: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|bit-equal|iters' gpurun_out/sanitize2_${tool}_32.log | tr '\n' ' ')"
done
for tool in memcheck synccheck racecheck; do
  FRB_VIRTUAL_ONLY=1 timeout 1500 $S --tool $tool --print-limit 50 python tools/sanitize_cluster.py 32 200 --check > gpurun_out/sanitize2_${tool}_32v.log 2>&1
  echo "virtual n=32 $tool rc=$?: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|bit-equal|iters' gpurun_out/sanitize2_${tool}_32v.log | tr '\n' ' ')"
done
