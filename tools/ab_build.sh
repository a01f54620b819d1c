# Build the library at git revision $1 into abl/$2.so (the working tree's
# build stays untouched):  bash tools/ab_build.sh HEAD A
set -e
REV=$1; TAG=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
WT=/tmp/w2l_ab_$TAG
rm -rf $WT; git -C $ROOT worktree prune; git -C $ROOT worktree add -f --detach $WT $REV >/dev/null
(cd $WT && python -m paper_1812_07625_b200._build >/dev/null)
mkdir -p $ROOT/abl; cp $WT/paper_1812_07625_b200/lib/libw2l_criterion.so $ROOT/abl/$TAG.so
git -C $ROOT worktree remove --force $WT
echo "abl/$TAG.so <- $REV"
