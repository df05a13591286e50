# Build ab/libls_A.so from the committed HEAD sources (the working tree's
# changes stashed), then the working tree's libls.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p ab
git stash -q
make -s -j16 paper_2107_03290_b200/libls.so > /dev/null 2>&1 || true
cp paper_2107_03290_b200/libls.so ab/libls_A.so
git stash pop -q
make -s -j16 paper_2107_03290_b200/libls.so > /dev/null 2>&1
echo built
