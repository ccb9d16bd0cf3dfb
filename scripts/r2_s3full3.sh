# session 3: host-mapped meta ring restored + stage-thread budget; c2, gpu tests, full bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3full3; mkdir -p $O
( time timeout 400 python bench.py --legs c2 --c2-decode 16 ) > $O/c2.log 2>&1; echo "rc=$?" >> $O/c2.log
( time timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
( time timeout 1500 python bench.py ) > $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
echo done
