DTANS_LIB=paper_2603_01915_b200/exp/libdtans_wc.so python bench.py --config rmat --reorder --steps 3 --no-cpu-baseline --no-cusparse 2>&1 | tail -2
DTANS_LIB=paper_2603_01915_b200/exp/libdtans_wc.so DTANS_LONG_SEG=4 python -m pytest tests/test_gpu.py -x -q -k "larger or long_slice" 2>&1 | tail -3
