timeout 1200 python -m pytest tests/test_gpu_summa.py -x -q -k "per_round" 2>&1 | grep -E "assert|Error|peak|ok=" | head -20
