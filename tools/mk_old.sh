# build libsgwg_old.so from HEAD (A/B baseline for tools/exp_ab.sh), then rebuild the working tree
set -e
git stash -q
python -m paper_2007_10196_b200.build > /dev/null
cp paper_2007_10196_b200/libsgwg.so paper_2007_10196_b200/libsgwg_old.so
git stash pop -q
touch paper_2007_10196_b200/csrc/kernels.cuh
python -m paper_2007_10196_b200.build > /dev/null
echo built
