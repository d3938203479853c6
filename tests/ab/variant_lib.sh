#!/usr/bin/env bash
# Same-box A/B builds (not a test): link libswarmsched_b200.so with ONE source rebuilt under extra nvcc flags.
#   bash tests/ab/variant_lib.sh <name> <file.cu> [-DMACRO=value ...]   ->  variants/<name>.so
# e.g. bash tests/ab/variant_lib.sh unroll4 replay_regions.cu -DRG_UNROLL=4
# then python tests/ab/region_ab.py variants/unroll4.so variants/base.so  (on a B200, through gpurun)
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
cd "$ROOT/paper_2509_26182_b200/csrc"
OBJ=${AB_OBJ_DIR:-/tmp/ss_ab_objs}
mkdir -p "$OBJ" "$ROOT/variants"
ARCH="-gencode arch=compute_100a,code=sm_100a"
FL="-O3 -lineinfo -fmad=false -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC"
name=$1; src=$2; shift 2
objs=""
for f in *.cu; do
  b=${f%.cu}
  if [ "$f" == "$src" ]; then
    nvcc $ARCH $FL "$@" -c "$f" -o "$OBJ/var_$b.o"; objs="$objs $OBJ/var_$b.o"
  else
    if [ ! -f "$OBJ/$b.o" ] || [ "$f" -nt "$OBJ/$b.o" ]; then nvcc $ARCH $FL -c "$f" -o "$OBJ/$b.o"; fi
    objs="$objs $OBJ/$b.o"
  fi
done
nvcc $ARCH -shared -o "$ROOT/variants/$name.so" $objs
echo "built variants/$name.so"
