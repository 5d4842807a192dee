# compute-sanitizer over tests/sanitize_cases.py; logs -> gpurun_out/san_*.log
python -m paper_2506_15155_b200.build > /dev/null 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for c in c1 pdl gather prefill; do
  for tool in memcheck racecheck synccheck; do
    extra=""; [ $tool = memcheck ] && extra="--leak-check no"
    timeout 900 $CS --tool $tool $extra --print-limit 20 python tests/sanitize_cases.py $c > gpurun_out/san_${c}_${tool}.log 2>&1
    echo "$c $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case .*: ok' gpurun_out/san_${c}_${tool}.log | tr '\n' ' ')"
  done
done
