# builds experimental library variants into paper_2310_03294_b200/variants/
set -e
mkdir -p paper_2310_03294_b200/variants
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  DA_BUILD_DIR=/tmp/da_build_$name DA_LIB_OUT=paper_2310_03294_b200/variants/lib_$name.so DA_BUILD_DEFINES="$defs" python paper_2310_03294_b200/build.py --force >/dev/null
  echo built $name
done
