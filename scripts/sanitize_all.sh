python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out; o=gpurun_out/sanitizer.txt; : > $o
for t in memcheck racecheck synccheck; do
  echo "== compute-sanitizer --tool $t python scripts/sanitize_small.py (round 1) ==" >> $o
  timeout 900 compute-sanitizer --tool $t python scripts/sanitize_small.py >> $o 2>&1
  echo >> $o
done
tail -40 $o
