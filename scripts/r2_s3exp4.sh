# session 3: reduce rewrite (pipelined items, fp32 8-partials), overload leg, c2 with the oversize page-out cache
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3exp4; mkdir -p $O
( time timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_observer.py -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
timeout 300 python scripts/exp_ops.py > $O/ops.jsonl 2>&1
( time timeout 900 python bench.py --legs overload ) > $O/overload.log 2>&1; echo "rc=$?" >> $O/overload.log
( time timeout 900 python bench.py --legs c2 --c2-decode 32 --model-ring-mib 8192 ) > $O/c2.log 2>&1; echo "rc=$?" >> $O/c2.log
echo done
