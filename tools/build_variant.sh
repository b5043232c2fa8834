# build paper_1103_4881_b200/libds_<name>.so with extra nvcc flags (tuning A/B):
#   bash tools/build_variant.sh t28 -DDS_GEN_STAGE_TARGET=28672 -DDS_GEN_CTAS=3 -DDS_GEN_MINB=3
name=$1; shift
cd "$(dirname "$0")/.." && /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC,-fvisibility=hidden -shared -Xptxas=-v "$@" -I include paper_1103_4881_b200/csrc/*.cu \
  -ldl -o paper_1103_4881_b200/libds_$name.so 2>&1 | grep -A2 "general_kernel" | grep -E "Used|spill"
