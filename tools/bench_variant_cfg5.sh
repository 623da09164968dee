cd "${GRAFT_REPO_ROOT:-.}"; mkdir -p gpurun_out/x5
for r in 1 2; do
timeout 300 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x5/lib$r.json 2>/dev/null
timeout 300 python -c "
import sys, runpy; sys.path.insert(0, '.')
from paper_1703_10119_b200 import api; api.load_library('tools/_ringvar/libhygro_MATRCP.so')
sys.argv = ['bench.py', '--config', 'cfg5', '--steps', '3', '--warmup', '3', '--no-cpu-baseline', '--no-e2e']
runpy.run_path('bench.py', run_name='__main__')" > gpurun_out/x5/var$r.json 2>gpurun_out/x5/var$r.err
done
