#!/bin/bash
# dev helper (CPU box): build tuning variants of the library side by side.
#   tools/build_variants.sh "name1|-DSFB_X=1" "name2|-DSFB_Y=2 -DSFB_Z=3" ...
# -> paper_2107_02671_b200/lib/var_<name>.so (run them with tools/run_variants.sh)
cd "$(dirname "$0")/../paper_2107_02671_b200/csrc"
for spec in "$@"; do
  name=${spec%%|*}; extra=${spec#*|}
  make -s -j8 BUILD=build_var_$name OUT=../lib/var_$name.so EXTRA="$extra" || exit 1
  rm -rf build_var_$name; echo "built var_$name ($extra)"
done
