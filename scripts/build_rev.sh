# usage: bash scripts/build_rev.sh <git-rev> <out.so>  -- build libpfac from another revision (A/B runs)
set -e
rev=$1; out=$2; tmp=$(mktemp -d)
git archive "$rev" paper_1811_10498_b200/csrc include | tar -x -C "$tmp"
srcs=$(ls $tmp/paper_1811_10498_b200/csrc/*.cu $tmp/paper_1811_10498_b200/csrc/*.cpp)
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC,-O2 -shared --cudart static -o "$out" $srcs
rm -rf "$tmp"
