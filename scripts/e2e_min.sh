python -m pytest tests/test_gpu_parity.py -q -k "pairs" 2>&1 | tail -2
for m in 16384 32768 65536 131072; do LSNIF_HOST_MIN_CHUNK=$m python scripts/e2e_tune.py 131072 | sed "s/^/min=$m /"; done
