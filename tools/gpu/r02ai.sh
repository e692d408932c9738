timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r02ai_test.txt
O=gpurun_out/sanitizer_r02b.txt
echo "# compute-sanitizer on the coalesced kernel (round 2 after the tensor-staged GEMV + warp-uniform issue changes, B200, tools/sanitize_target.py)" > $O
for w in step resident; do for t in memcheck racecheck synccheck; do
  echo "## san_${w}_${t}" >> $O
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_target.py $w 2>&1 | grep -E "ok$|SUMMARY|Invalid|Error|error" | head -20 >> $O
  echo "rc=${PIPESTATUS[0]}" >> $O
done; done
for i in 1 2; do timeout 200 python tools/ab_held.py _ab/prev/libgmx_exec.so >> gpurun_out/r02ai.txt 2>&1; timeout 200 python tools/ab_held.py >> gpurun_out/r02ai.txt 2>&1; done
