# session 3: small-capture launch without shared-memory speculation, one barrier fewer on the ballot path
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3small; mkdir -p $O
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_gpu_vllm.py ) > $O/pytest.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 --reps 7 --out $O/dec_idle.json > $O/dec_idle.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 16 --sizes-kb 1024,4096,32768,114688 --row-bytes 8192 --reps 7 --out $O/big_idle.json > $O/big_idle.log 2>&1
timeout 300 python scripts/exp_sweep.py --n 32 --batch 16 --sizes-kb 128,448 --row-bytes 8192 --busy-d2h --out $O/dec_busy.json > $O/dec_busy.log 2>&1
( time timeout 600 python bench.py --legs value --steps 20 ) > $O/bench_value.log 2>&1
echo done
