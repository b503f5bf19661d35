# usage: bash tools/ab_build.sh REV OUT.so — build libjanus_b200.so of git revision REV into OUT.so
# (A/B timing of two kernel versions in one gpurun call: JANUS_LIB=OUT.so python ...)
set -e
REV=$1; OUT=$2
D=$(mktemp -d)
git archive "$REV" paper_2512_13525_b200/csrc include | tar -x -C "$D"
SRCS=$(ls $D/paper_2512_13525_b200/csrc/*.cu $D/paper_2512_13525_b200/csrc/*.cpp)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -Xcompiler -fopenmp -I$D/include -o "$OUT" $SRCS -lgomp
rm -rf "$D"
