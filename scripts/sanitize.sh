# compute-sanitizer over the fused pass (C1, C4), a multigrid solve and the
# loop helpers: memcheck, racecheck (shared-memory hazards), synccheck
# (barrier misuse); logs -> gpurun_out/sanitizer_<tool>_<what>.txt
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for what in pass solve; do
    timeout 1500 $CS --tool $tool --error-exitcode 17 python scripts/sanitize.py $what \
      > gpurun_out/sanitizer_${tool}_${what}.txt 2>&1
    echo "$tool $what rc=$? $(tail -1 gpurun_out/sanitizer_${tool}_${what}.txt)"
  done
done
timeout 1500 $CS --tool memcheck --error-exitcode 17 python -m pytest -q -x tests/test_gpu_loop.py \
  > gpurun_out/sanitizer_memcheck_loop.txt 2>&1; echo "memcheck loop rc=$? $(tail -1 gpurun_out/sanitizer_memcheck_loop.txt)"
