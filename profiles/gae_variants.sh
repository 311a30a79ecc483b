# Round-1 GAE experiment driver (results: profiles/r1_gae_variants.txt). The GAE_STAGES /
# GAE_MIN_BLOCKS / GAE_RECOMPUTE_D macros it sets lived in an experimental csrc/gae.cu that was
# reverted after no variant beat the shipped kernel; with today's gae.cu the -D flags are no-ops.
set -x
cd $GRAFT_REPO_ROOT
for cfg in "2 2 0" "2 3 1" "3 2 0" "3 2 1" "2 2 1"; do
  set -- $cfg
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Iinclude -DGAE_STAGES=$1 -DGAE_MIN_BLOCKS=$2 -DGAE_RECOMPUTE_D=$3 -c paper_2603_18464_b200/csrc/gae.cu -o paper_2603_18464_b200/_build/gae.o
  touch paper_2603_18464_b200/_build/gae.o
  python -m paper_2603_18464_b200.build > /dev/null
  echo "VARIANT S=$1 B=$2 R=$3"
  timeout 120 python profiles/gae_bench.py 4096 16384 65536
  timeout 120 python profiles/gae_bench.py 65536
  timeout 300 python -m pytest -q -x -m gpu -p no:cacheprovider -k "gae or GAE or normaliz" tests 2>&1 | tail -1
done
