set -x
timeout 1800 python -m pytest tests/ -m gpu -q -p no:cacheprovider -x 2>&1 | tail -3
timeout 900 python scripts/cfg_run.py cfg4 --capped 4 > gpurun_out/r02_cfg4_1gpu_capped.json 2> gpurun_out/cfg4.err
timeout 900 python scripts/cfg_run.py cfg5 --capped 3 > gpurun_out/r02_cfg5_1gpu_capped.json 2> gpurun_out/cfg5.err
timeout 600 python scripts/dense_shapes.py 2097152 16,48,80,192 > gpurun_out/r02_dense_shapes_2M.json 2> gpurun_out/r02_dense_shapes_2M.err
python - <<'PY'
import json
for f in ["gpurun_out/r02_cfg4_1gpu_capped.json","gpurun_out/r02_cfg5_1gpu_capped.json"]:
    d=json.load(open(f))
    for v in d["capped"]:
        print(f, v["variant"], {k: round(x["ms_per_iteration_median"],1) for k,x in v["per_stage_from_records"].items()})
PY
