# builds the committed HEAD's native library into exp/head.so (for tools/ab_lib.sh)
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/wt_head && git worktree add -q /tmp/wt_head HEAD
(cd /tmp/wt_head && python paper_2504_06182_b200/build_native.py > /tmp/wt_head_build.log 2>&1)
cp /tmp/wt_head/paper_2504_06182_b200/lib/librecon_b200.so exp/head.so
git worktree remove --force /tmp/wt_head
