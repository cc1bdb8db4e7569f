# compile-time variants of libnsl for the perf sweep (NSL_LIB selects one at run time)
set -e
cd "$(dirname "$0")/.."
for mb in 1 4 5 6; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
       -DNSL_MINB=$mb -o /tmp/libnsl_mb$mb.so paper_2604_03748_b200/csrc/*.cu &
done
wait
