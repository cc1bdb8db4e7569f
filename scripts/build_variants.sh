# compile-time variants of libnsl for the perf sweep (NSL_LIB selects one at run time)
set -e
cd "$(dirname "$0")/.."
for mb in ${MBS:-5}; do for th in 8; do for st in 0 1; do for pw in 0; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
       -DNSL_MINB=$mb -DNSL_TILEH=$th -o /tmp/libnsl_mb${mb}_t${th}_s${st}.so \
       paper_2604_03748_b200/csrc/*.cu 2>/dev/null &
done; done; done; done
wait
