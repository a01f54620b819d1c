# Build the WORKING TREE's library with extra nvcc flags into abl/$1.so:
#   bash tools/ab_flags.sh spl8 -DW2L_SPL=8
set -e
TAG=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/w2l_abf_$TAG
rm -rf $WT; mkdir -p $WT
cp -r $ROOT/paper_1812_07625_b200 $ROOT/include $WT/
rm -rf $WT/paper_1812_07625_b200/lib $WT/paper_1812_07625_b200/build
(cd $WT && W2L_EXTRA_NVCC_FLAGS="$*" python -m paper_1812_07625_b200._build >/dev/null)
mkdir -p $ROOT/abl; cp $WT/paper_1812_07625_b200/lib/libw2l_criterion.so $ROOT/abl/$TAG.so
echo "abl/$TAG.so <- working tree + $*"
