# Diagnosis builds of one kernel source (SRC=umma_tma default, or ops, ...) with experiment macros,
# each linked into tools/probes/_build/<name>/libpbkd_b200.so (product objects
# otherwise).  Usage: tools/probes/build_variants.sh name=-DMACRO ...
set -e
SRC=${SRC:-umma_tma}
R=$(cd "$(dirname "$0")/../.." && pwd)
P=$R/paper_2012_03096_b200
make -s -C $P -j16
JSON_INC=$(python3 -c "import os,site;[print(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann')) for p in site.getsitepackages() if os.path.isdir(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann'))]" | head -1)
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  out=$R/tools/probes/_build/$name; mkdir -p $out
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC \
    -Xcompiler -ffp-contract=off -I$P/include -I$R/include -I$JSON_INC --expt-relaxed-constexpr $flags \
    -c $P/csrc/$SRC.cu -o $out/$SRC.o
  objs=$(ls $P/build/obj/*.o | grep -v "/$SRC.o\$")
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libpbkd_b200.so $objs $out/$SRC.o -lcudart
  rm -f $out/$SRC.o
  echo "built $name ($flags)"
done
