# session 3: gated eager captures (c2 + overload legs, new gpu test), then the
# vLLM serving sweep up to 256 req/s (configs[3])
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3vllm; mkdir -p $O
( time timeout 600 python -m pytest tests/test_gpu_observer.py -x -q -p no:cacheprovider ) > $O/pytest_observer.log 2>&1
( time timeout 900 python bench.py --legs c2 --c2-decode 32 --model-ring-mib 8192 ) > $O/c2.log 2>&1; echo "rc=$?" >> $O/c2.log
( time timeout 900 python bench.py --legs overload ) > $O/overload.log 2>&1; echo "rc=$?" >> $O/overload.log
RATES=1,4,16,64,256 N=128 VT=1500 bash scripts/vllm_ab.sh > $O/vllm_summary.txt 2>&1
cp gpurun_out/vllm_*.log $O/ 2>/dev/null
echo done
