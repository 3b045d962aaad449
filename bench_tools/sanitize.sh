# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tiny invocations of every
# kernel family (bench_tools/sanitize_case.py). usage: bash bench_tools/sanitize.sh TAG
T=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for w in attn_bf16 attn_fp32 loss tree rope; do
    echo "== $tool $w" >> gpurun_out/${T}_sanitize.txt
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python bench_tools/sanitize_case.py $w >> gpurun_out/${T}_sanitize.txt 2>&1
    echo "rc=$?" >> gpurun_out/${T}_sanitize.txt
  done
done
grep -E "^== |rc=|ERROR SUMMARY" gpurun_out/${T}_sanitize.txt | paste - - - | head -40
