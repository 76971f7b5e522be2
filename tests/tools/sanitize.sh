# compute-sanitizer over the kernels: memcheck, racecheck
# (shared-memory hazards), synccheck (barrier misuse), initcheck (reads of
# uninitialised device memory) on tests/tools/sanitize_run.py, float64 and
# tf32 modes.  usage: bash tests/tools/sanitize.sh [tag]
# NOTE: compute-sanitizer is closed on the graft GPU pool ("Tracing, checks and switches"); this script is for other machines.
TAG=${1:-san}
for tool in memcheck racecheck synccheck initcheck; do
  for dt in f64 tf32; do
    GEVO_B200_DTYPE=$dt timeout 600 compute-sanitizer --tool $tool --print-limit 20 \
      python tests/tools/sanitize_run.py > gpurun_out/${TAG}_${tool}_${dt}.log 2>&1
    echo "$tool $dt rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|opcases' gpurun_out/${TAG}_${tool}_${dt}.log | tr '\n' ' ')"
  done
done
