# Build A/B variants of libnsl.so HERE (no GPU needed) into abl/ (git-ignored, shipped by gpurun):
#   VARIANTS="base:;hz0:-DNSL_HZ=0" bash scripts/ab_local.sh
# Each variant recompiles the translation units in TUS (default: march.cu) with its flags and links
# them with the default objects of the other units (paper_2604_03748_b200/lib/obj, from build()).
set -e
cd "$(dirname "$0")/.."
python -c "import paper_2604_03748_b200 as n; n.build()"
mkdir -p abl
IFS=';' read -ra VS <<< "${VARIANTS}"
TUS=${TUS:-march}
OBJ=paper_2604_03748_b200/lib/obj
for v in "${VS[@]}"; do
  name="${v%%:*}"; flags="${v#*:}"
  (
    mkdir -p abl/obj_$name
    objs=""
    for o in $OBJ/*.o; do
      b=$(basename $o .o)
      if [[ " $TUS " == *" $b "* ]]; then
        nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC $flags \
             -c -o abl/obj_$name/$b.o paper_2604_03748_b200/csrc/$b.cu
        objs="$objs abl/obj_$name/$b.o"
      else
        objs="$objs $o"
      fi
    done
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o abl/libnsl_$name.so $objs
    echo "built abl/libnsl_$name.so ($flags)"
  ) &
done
wait
