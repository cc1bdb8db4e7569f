# Checked build (device asserts on every computed volume / mask / lattice index, NSL_CHECK=1)
# and the GPU test suite against it; a failed assert aborts the kernel and fails the test.
set -e
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -cudart static \
     -DNSL_CHECK=1 -o /tmp/libnsl_checked.so paper_2604_03748_b200/csrc/*.cu
NSL_LIB=/tmp/libnsl_checked.so timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider
