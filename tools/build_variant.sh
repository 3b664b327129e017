#!/bin/bash
# Build a variant of the library with extra -D defines (A/B experiments):
#   tools/build_variant.sh NAME "DEF1 DEF2=3"  ->  tools/var/NAME/libvc3_b200.so
# Objects of unchanged translation units are copied from lib/obj first.
set -e
cd "$(dirname "$0")/.."
out=tools/var/$1
mkdir -p $out/obj
cp -p paper_2003_02633_b200/lib/obj/*.o $out/obj/ 2>/dev/null || true
touch paper_2003_02633_b200/csrc/vc3_fused_as.cu -r paper_2003_02633_b200/csrc/vc3_fused_as.cu
rm -f $out/obj/vc3_fused_as.o
VC3_BUILD_OUT=$out VC3_BUILD_DEFINES="$2" python -c "from paper_2003_02633_b200 import _build; _build.build()"
echo $out/libvc3_b200.so
