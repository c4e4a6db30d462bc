o=gpurun_out/sanitizer.txt; : > $o
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --error-exitcode 3 python tools/sanitize.py > /tmp/san_$t.log 2>&1
  echo "$t rc=$?: $(grep 'sanitize driver done' /tmp/san_$t.log)" >> $o
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" /tmp/san_$t.log | tail -1 | sed "s/^/$t: /" >> $o
  grep -m5 "Invalid\|Race\|Barrier\|Uninitialized" /tmp/san_$t.log | sed "s/^/$t: /" >> $o
done
