mkdir -p gpurun_out
python - <<'PY' > gpurun_out/ab1_ulps.txt 2>&1
import numpy as np, torch
from paper_2509_13230_b200 import fastmaxent as fm
rng=np.random.default_rng(0)
def u(a,b): return np.abs(a.view(np.int64)-b.view(np.int64))
x=np.exp(rng.uniform(-700,700,4_000_000)); y=fm.debug_eval(0,torch.from_numpy(x)).cpu().numpy(); d=u(y,np.log(x)); print('log', d.max(), (d==0).mean(), np.bincount(d)[:5])
x=np.exp(rng.uniform(np.log(1e-300),np.log(1e300),4_000_000)); y=fm.debug_eval(1,torch.from_numpy(x)).cpu().numpy(); d=u(y,np.log1p(x)); print('log1p', d.max(), (d==0).mean(), np.bincount(d)[:5])
x=rng.uniform(0,2,4_000_000); y=fm.debug_eval(1,torch.from_numpy(x)).cpu().numpy(); d=u(y,np.log1p(x)); print('log1p[0,2]', d.max(), (d==0).mean(), np.bincount(d)[:5])
k=np.arange(0,2**32,997,dtype=np.int64); uu=(k+0.5)*2.0**-32; y=fm.debug_eval(2,torch.from_numpy(k.astype(np.float64))).cpu().numpy(); d=u(y,-np.log(uu)); print('E', d.max(), (d==0).mean(), np.bincount(d)[:5])
PY
cat gpurun_out/ab1_ulps.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab1_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/ab1_pytest.log
for c in 2 3 4; do AB_VARIANTS="head base cs" AB_ARGS="--config $c" bash scripts/ab.sh; done 2>&1 | tee gpurun_out/ab1.txt
