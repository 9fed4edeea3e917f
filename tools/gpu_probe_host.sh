# host facts of the GPU box: memory, cores, pinned-allocation ceiling, numba, reference import
set -x
nproc; free -g; cat /sys/fs/cgroup/memory.max 2>/dev/null; lscpu | grep -E "Model name|Socket|Thread|Core"
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python - <<'PY'
import time, torch
for gb in (8, 32, 64, 100):
    t = time.time()
    try:
        x = torch.empty(gb << 27, dtype=torch.float64, pin_memory=True)
        print("pinned", gb, "GB ok", round(time.time() - t, 2), "s"); del x
    except Exception as e:
        print("pinned", gb, "GB FAIL", e); break
PY
PYTHONPATH=baseline/_ref python -c "import trihalo, numba; print('reference import ok', numba.__version__)"
