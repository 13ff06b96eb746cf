# trace variant (cycles/tile per epilogue phase) + A/B bench of the in-tree library
SURGE_LIB=varlib/tr.so PYTHONPATH=. timeout 300 python scripts/att_trace.py 2>&1 | grep ATT_TRACE | awk '!seen[$5]++' | sort -k5n | head -12
bash scripts/gpu_ab.sh
