cd $GRAFT_REPO_ROOT
for v in A B A B; do echo "== lib $v"; HB200_LIB=$PWD/paper_2209_05819_b200/lib/libhb200_$v.so timeout 300 python tools/gemm_bench.py 5 2>&1 | grep -E "8192x|32768x32768x120|120x32768|128x65536|65536x65536x120|20000x"; done
