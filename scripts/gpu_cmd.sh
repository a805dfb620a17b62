mkdir -p gpurun_out
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('l2', p.L2_cache_size)
from cuda.bindings import runtime as rt
print(rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize, 0), rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0))" 2>&1 | tail -3
AB_RUNS=$'base4;;--config 4\np40;FM_L2_PERSIST=40;--config 4\np80;FM_L2_PERSIST=80;--config 4' AB_STEPS=5 bash scripts/abx.sh 2>&1 | tee gpurun_out/ab41.txt
