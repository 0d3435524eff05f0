timeout 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "tensor_cores or gram" 2>&1 | tail -3
python scripts/tc_exp.py
