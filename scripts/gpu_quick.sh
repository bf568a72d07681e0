set -x
python scripts/dbg_infer.py
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "not infer" 2>&1 | tail -30
