for i in 1 2 3; do
DTANS_LONG_SEG=4 python -m pytest tests/test_gpu.py -x -q -k "larger_matrices" 2>&1 | grep -E "passed|failed|Error|assert" | head -5
DTANS_LONG_SEG=4 DTANS_TASK_GMEM=1 python -m pytest tests/test_gpu.py -x -q -k "larger_matrices" 2>&1 | grep -E "passed|failed|Error" | head -3
done
