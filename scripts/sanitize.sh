# Sanitizer runs of the lock-free device<->host protocol.
# Builds tests/native/stress_protocol.cu against the library sources twice:
#   /tmp/stress_plain  -lineinfo, for compute-sanitizer memcheck/racecheck/synccheck
#   /tmp/stress_tsan   host code (library + driver) with -fsanitize=thread
# and runs them; logs under gpurun_out/sanitize/ (copied to profiles/sanitizer/).
cd ${GRAFT_REPO_ROOT:-$(dirname $0)/..}
O=gpurun_out/sanitize; mkdir -p $O
C=paper_2605_11093_b200/csrc
SRC="tests/native/stress_protocol.cu $C/ring2.cu $C/stager.cu $C/sink.cpp"
FL="-gencode arch=compute_100a,code=sm_100a -O2 -lineinfo -std=c++17 --expt-relaxed-constexpr -Iinclude -lz -lpthread -lcuda"
nvcc $FL -Xcompiler -fPIC,-pthread -o /tmp/stress_plain $SRC > $O/build_plain.log 2>&1 || echo "plain build failed" >> $O/build_plain.log
nvcc $FL -Xcompiler -fsanitize=thread,-fPIC,-pthread,-g -ltsan -o /tmp/stress_tsan $SRC > $O/build_tsan.log 2>&1 || echo "tsan build failed" >> $O/build_tsan.log
N=${STRESS_N:-1500}
( time timeout 300 /tmp/stress_plain $N 1 ) > $O/plain_1ring.log 2>&1; echo "rc=$?" >> $O/plain_1ring.log
( time timeout 300 /tmp/stress_plain $N 2 ) > $O/plain_2rings.log 2>&1; echo "rc=$?" >> $O/plain_2rings.log
( time timeout 300 /tmp/stress_plain $N 2 1 ) > $O/plain_2rings_sealed.log 2>&1; echo "rc=$?" >> $O/plain_2rings_sealed.log
for tool in memcheck racecheck synccheck; do
  ( time timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 /tmp/stress_plain 300 1 ) > $O/cs_$tool.log 2>&1
  echo "rc=$?" >> $O/cs_$tool.log
  ( time timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 /tmp/stress_plain 300 1 1 ) > $O/cs_${tool}_sealed.log 2>&1
  echo "rc=$?" >> $O/cs_${tool}_sealed.log
done
( time TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 report_signal_unsafe=0" timeout 900 /tmp/stress_tsan 600 2 ) > $O/tsan.log 2>&1
echo "rc=$?" >> $O/tsan.log
( time TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 report_signal_unsafe=0" timeout 900 /tmp/stress_tsan 600 2 1 ) > $O/tsan_sealed.log 2>&1
echo "rc=$?" >> $O/tsan_sealed.log
