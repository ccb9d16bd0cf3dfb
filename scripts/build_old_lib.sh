# Build the library of a git revision as an experiment variant
# (_lib/libring2_<tag>.so, loaded with TF_LIB_VARIANT=<tag>) for same-box
# A/B runs against the working tree. usage: scripts/build_old_lib.sh REV TAG
set -e
cd $(dirname $0)/..
REV=$1; TAG=$2; T0=$(mktemp -d); T=$T0/pkg/x
mkdir -p $T/csrc $T0/pkg/include
for f in ring2.cu stager.cu sink.cpp ring2_core.h ring2_internal.h crc32_fast.h; do
  git show $REV:paper_2605_11093_b200/csrc/$f > $T/csrc/$f 2>/dev/null || true
done
git show $REV:include/ring2.h > $T0/pkg/include/ring2.h
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3,-pthread -I $T0/pkg/include"
for f in ring2.cu stager.cu sink.cpp; do nvcc $FL -c $T/csrc/$f -o $T/${f%.*}.o; done
nvcc -shared -gencode arch=compute_100a,code=sm_100a $T/*.o -o paper_2605_11093_b200/_lib/libring2_$TAG.so -Xcompiler -pthread -lpthread -lz
rm -rf $T0
echo built paper_2605_11093_b200/_lib/libring2_$TAG.so
