# A/B of capture-kernel variants with scripts/exp_sweep.py (per-launch us)
summ() { python -c "
import sys,json
out=[]
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); out.append(f\"{d['mib']}:{d['capture_us']:.1f}\")
    elif 'Error' in l or 'error' in l: out.append(l.strip()[:200])
print(' '.join(out))"; }
for v in ${VARIANTS:-""}; do
  [ "$v" = "product" ] && v=""
  echo -n "variant '${v:-product}': "
  TF_LIB_VARIANT=$v timeout 200 python scripts/exp_sweep.py --sizes-mib ${SIZES:-1,8,32,112,224} --reps 5 --out gpurun_out/sw.json 2>&1 | summ
done
