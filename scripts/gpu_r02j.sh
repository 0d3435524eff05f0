python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r02j.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_r02j.log
timeout 900 python scripts/cfg_run.py cfg4 --capped 4 > gpurun_out/r02_cfg4_capped_c.json 2> gpurun_out/r02_cfg4_capped_c.log
timeout 600 python scripts/cfg_run.py cfg2 --capped 40 --pinvit 20 --variants mplobpcg-schol,dlobpcg-dchol > gpurun_out/r02_cfg2_capped_c.json 2> gpurun_out/r02_cfg2_capped_c.log
