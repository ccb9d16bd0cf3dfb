# session 3: warp-local keep scan for <= 32 keep units
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3tiny; mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 --sealed --reps 9 --out $O/dec_sealed.json > $O/dec_sealed.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 --sealed --busy-d2h --reps 9 --out $O/dec_sealed_busy.json > $O/dec_sealed_busy.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 1024,32768,114688 --row-bytes 8192 --sealed --reps 7 --out $O/big_sealed.json > $O/big_sealed.log 2>&1
echo done
