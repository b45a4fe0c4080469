O=gpurun_out/san; mkdir -p $O
timeout 300 python tools/sanitize_driver.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -1 $O/plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --kernel-name kns=fsdp --error-exitcode 9 --print-limit 50 python tools/sanitize_driver.py > $O/$tool.log 2>&1; echo "$tool rc=$?"
  tail -4 $O/$tool.log
done
