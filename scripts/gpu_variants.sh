# run scripts/att_trace.py against each varlib/*.so
for so in varlib/*.so; do
  echo "== $so"
  SURGE_LIB=$so PYTHONPATH=. timeout 300 python scripts/att_trace.py 2>&1 | grep ATT_TRACE | awk '!seen[$5]++' | sort -k5n | head -12
done
