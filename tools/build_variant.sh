#!/bin/bash
# experiment build: tools/build_variant.sh <name> [-D...]: recompiles law_euler.cu with the extra flags on top of
# the cached objects of the base build (STROM_OBJ_DIR=build/obj_base python -m paper_2305_15661_b200.build --force)
# and links abso/<name>.so (A/B with tools/ab2.sh)
name=$1; shift
rm -rf build/obj_$name; cp -r build/obj_base build/obj_$name; mkdir -p abso
STROM_OBJ_DIR=build/obj_$name STROM_ONLY_UNITS=${UNITS:-law_euler.cu} STROM_NVCC_EXTRA="$*" STROM_SO_OUT=abso/$name.so \
  python -m paper_2305_15661_b200.build --force
