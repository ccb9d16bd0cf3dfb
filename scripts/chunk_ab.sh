for c in 16 8 32 16 8 32; do echo -n "chunk $c: "; TF_CAP_CHUNK_KB=$c VARIANTS="product" bash scripts/bench_ab.sh; done
for c in 16 8; do echo "chunk $c sweep:"; TF_CAP_CHUNK_KB=$c timeout 300 python scripts/exp_sweep.py --sizes-kb 128,448,1024,4096 --n 32 2>&1 | cut -c1-48; done
