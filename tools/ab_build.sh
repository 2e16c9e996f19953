#!/bin/bash
# Build the csrc + include of git revision $1 into $2 (A/B timing on one GPU box).
set -e
REV=$1; OUT=$2
TMP=$(mktemp -d)
git -C /root/repo archive "$REV" paper_2306_02272_b200/csrc include | tar -x -C "$TMP"
python -m paper_2306_02272_b200.build --csrc "$TMP/paper_2306_02272_b200/csrc" --inc "$TMP/include" --out "$OUT"
rm -rf "$TMP"
