python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
python bench.py --no-cpu-baseline > gpurun_out/bench.log 2> gpurun_out/bench.err; echo rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["mttkrp_ms_per_mode"], d["e2e"]["ms_per_step"], d["cp_apr"]["s_per_outer_iteration"], d["cp_apr"]["phi_ms_avg"])
PY
