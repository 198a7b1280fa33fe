cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/c1_probe.py 1024,4096,16384,65536
python tools/polymul_sizes.py
python tools/polymul_probe.py 50
python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); ex=d['extras']
print(d['ms_per_step'], d['roofline']['per_kernel_ms']); print(ex['config1_kyber7_fwd_4096']); print({k:round(v['products_per_s']/1e9,3) for k,v in ex['config2_kyber_polymul_65536_fused'].items()}); print({k:v['ms'] for k,v in ex['config3_dilithium_roundtrip_65536'].items()})"
