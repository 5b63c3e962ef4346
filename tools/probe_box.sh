set -x
nproc; free -g; lscpu | head -25; nvidia-smi topo -m; cat /proc/meminfo | head -5
python - <<'PY'
import time, os, numpy as np, sys
sys.path.insert(0, '.')
import oracle
n=1024
f=np.random.default_rng(0).standard_normal((n,n,n))
for th in (16, len(os.sched_getaffinity(0))):
    oracle.set_threads(th, 'ref')
    t=time.perf_counter(); oracle.poisson_solve(f,'ref'); print('ref threads',th,'1024^3 s',time.perf_counter()-t, flush=True)
import scipy.fft as sf
t=time.perf_counter(); F=sf.rfftn(f, workers=len(os.sched_getaffinity(0))); u=sf.irfftn(F, s=f.shape, workers=len(os.sched_getaffinity(0))); print('scipy all', time.perf_counter()-t, flush=True)
PY
