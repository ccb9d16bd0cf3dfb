# session 3: eager kernel loading (lazy-loading deadlock), device timelines per staging mode, all gpu tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3preload; mkdir -p $O
timeout 300 python scripts/exp_timeline.py --steps 3 --modes copy-engine --no-flush --out $O/noflush > $O/noflush.jsonl 2> $O/noflush.err; echo "rc=$?" >> $O/noflush.err
timeout 900 python scripts/exp_timeline.py --steps 4 --modes off,copy-engine,mapped --out $O/timeline > $O/timeline.jsonl 2> $O/timeline.err; echo "rc=$?" >> $O/timeline.err
( time timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider ) > $O/pytest.log 2>&1
echo done
