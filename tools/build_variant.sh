#!/bin/bash
# Build a variant of the library with extra -D defines (A/B experiments):
#   tools/build_variant.sh NAME "DEF1 DEF2=3" [full]  ->  tools/var/NAME/libvc3_b200.so
# Without "full", objects of the other translation units are copied from
# lib/obj and only vc3_fused_as.cu is recompiled.
set -e
cd "$(dirname "$0")/.."
out=tools/var/$1
rm -rf $out; mkdir -p $out/obj
if [ "$3" != "full" ]; then
  cp -p paper_2003_02633_b200/lib/obj/*.o $out/obj/ 2>/dev/null || true
  printf '%s' "$2" > $out/obj/defines.txt
  rm -f $out/obj/vc3_fused_as.o
fi
VC3_BUILD_OUT=$out VC3_BUILD_DEFINES="$2" python -c "from paper_2003_02633_b200 import _build; _build.build()"
echo $out/libvc3_b200.so
