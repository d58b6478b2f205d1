python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out; o=gpurun_out/sanitizer.txt; : > $o
for t in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $t python scripts/sanitize_small.py (round 2) ==" >> $o
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_small.py >> $o 2>&1
  echo >> $o
done
echo "== compute-sanitizer --tool memcheck python -m pytest tests -m gpu (round 2) ==" >> $o
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests -m gpu -x -q -p no:cacheprovider >> $o 2>&1
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed|mismatches [1-9]" $o
