# session 3 final gate on the last commit: all gpu tests, smoke, default bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3gate; mkdir -p $O
( time timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 1500 python bench.py --steps 20 --warmup 3 ) > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
echo done
