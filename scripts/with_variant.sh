#!/bin/bash
# scripts/with_variant.sh TAG cmd...  -- run cmd with scratch_libs/libhbmc_TAG.so
# in place of the in-tree library (A/B experiments on the GPU box), then
# restore the default build.
set -u
tag=$1; shift
lib=paper_1908_00741_b200/libhbmc_b200.so
cp -p "$lib" "$lib.default"
cp "scratch_libs/libhbmc_$tag.so" "$lib"
touch -r "$lib.default" "$lib"   # keep the mtime so the package does not rebuild
"$@"
rc=$?
mv "$lib.default" "$lib"
exit $rc
