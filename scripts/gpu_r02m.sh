python -m pytest tests -m gpu -q -p no:cacheprovider -k "ks" > gpurun_out/pytest_ks.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ks.log
timeout 900 python scripts/cfg_run.py cfg5 --capped 3 > gpurun_out/r02_cfg5_capped.json 2> gpurun_out/r02_cfg5_capped.log
timeout 900 python scripts/cfg_run.py ks64 --full --variants mplobpcg-schol,dlobpcg-dchol > gpurun_out/r02_ks64_full.json 2> gpurun_out/r02_ks64_full.log
