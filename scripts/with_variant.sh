# run a command with a variant build of libgpbbmm.so swapped in (diagnostics):
#   bash scripts/with_variant.sh scripts/variants/lib_x.so python scripts/kv_once.py ...
set -e
L=paper_1903_08114_b200/_lib/libgpbbmm.so
cp "$L" /tmp/libgpbbmm.orig.so
cp "$1" "$L"
shift
"$@" || true
cp /tmp/libgpbbmm.orig.so "$L"
