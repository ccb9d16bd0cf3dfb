# session 3: speculative first batch for per-token reductions
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3rspec; mkdir -p $O
( time timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_capture.py -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
timeout 300 python scripts/exp_ops.py > $O/ops.jsonl 2>&1
echo done
