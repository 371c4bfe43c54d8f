#!/bin/bash
# A/B timing of alternative builds of libwlp_b200.so (tools/_variants/*.so, git-ignored):
# each is copied into place and timed with tools/time_cfg.py on the same box.
#   bash tools/ab_variants.sh OUT.txt SPEC...
out=$1; shift
cp paper_1501_01405_b200/libwlp_b200.so /tmp/libwlp_current.so
for v in tools/_variants/*.so; do
  cp "$v" paper_1501_01405_b200/libwlp_b200.so
  echo "== $(basename $v)" >> "$out"
  python tools/time_cfg.py "$@" >> "$out" 2>&1
done
cp /tmp/libwlp_current.so paper_1501_01405_b200/libwlp_b200.so
