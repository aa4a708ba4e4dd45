python - <<'PY'
import torch
p=torch.cuda.get_device_properties(0); print("L2", p.L2_cache_size)
try:
    from cuda.bindings import runtime as rt
except Exception:
    from cuda import cudart as rt
for a in ["cudaDevAttrMaxPersistingL2CacheSize","cudaDevAttrMaxAccessPolicyWindowSize","cudaDevAttrL2CacheSize"]:
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr,a),0))
PY
for v in 0 1; do echo "L2KEEP=$v"; KRB_L2KEEP=$v python tools/iter_time.py --config c1 c2 2>&1 | tail -2; KRB_L2KEEP=$v KRB_PHASE_PROF=1 python tools/iter_time.py --config c2 --phases 2>&1 | tail -1; done
