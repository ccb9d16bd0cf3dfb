# A/B of capture-kernel knobs with scripts/exp_sweep.py (per-launch us)
summ() { python -c "
import sys,json
out=[]
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); out.append(f\"{d['mib']}:{d['capture_us']:.1f}\")
print(' '.join(out))"; }
for v in "" trace_abl64 ""; do echo -n "variant '${v:-product}': "; TF_LIB_VARIANT=$v timeout 200 python scripts/exp_sweep.py --sizes-mib 1,8,32,112,224 --reps 5 --out gpurun_out/sw.json 2>&1 | summ; done
