DTANS_VERBOSE=1 python -m pytest tests/test_gpu.py -x -q -k "config1" 2>&1 | grep -v "^$" | tail -30
