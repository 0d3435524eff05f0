mkdir -p gpurun_out
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_r02b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_r02b.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r02b.log
timeout 900 python scripts/cfg_run.py cfg2 --capped 40 --pinvit 40 --full --variants mplobpcg-schol > gpurun_out/r02_cfg2.json 2> gpurun_out/r02_cfg2.log
timeout 900 python scripts/cfg_run.py cfg4 --capped 8 > gpurun_out/r02_cfg4_capped.json 2> gpurun_out/r02_cfg4_capped.log
