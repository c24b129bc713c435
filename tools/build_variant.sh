# Build an alternative libtsg (variants/libtsg_<name>.so) with extra nvcc
# flags, for A/B timing with tools/exp_variants.sh (TSG_LIB selects it).
#   bash tools/build_variant.sh <name> "<-DFLAG=...>"
set -e
name=$1; extra=${2:-}
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/variants"
make -s -j8 -C "$root/paper_1804_00695_b200/csrc" EXTRA="$extra" BUILD="$root/variants/build_$name" \
     OUT="$root/variants/libtsg_$name.so"
