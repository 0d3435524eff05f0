set -x
nproc > gpurun_out/host.txt; lscpu >> gpurun_out/host.txt 2>&1; free -g >> gpurun_out/host.txt
nvidia-smi >> gpurun_out/host.txt
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r02a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02a.log
python scripts/envelope_device.py > gpurun_out/envelope_device.json 2> gpurun_out/envelope_device.log
python -c "
import json, bench
res, wall, info, conc = bench.reference_full_solves('cfg1', 'mplobpcg-schol', 6)
print(json.dumps(bench.reference_summary('cfg1', 'mplobpcg-schol', res, wall, info, conc)))
" > gpurun_out/ref_full_6.json 2>&1
