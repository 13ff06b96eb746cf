for so in varlib/split1.so varlib/split0.so; do echo "== $so"; SURGE_LIB=$so PYTHONPATH=. timeout 900 python scripts/parity_margin.py; done
