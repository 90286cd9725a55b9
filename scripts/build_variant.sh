#!/bin/bash
# Build a library variant with some csrc files taken from a git revision:
#   bash scripts/build_variant.sh <name> <rev> <file.cu> [file.cu ...]   -> variants/<name>.so
set -e
name=$1; rev=$2; shift 2
D=paper_2110_10221_b200/build_var_$name
rm -rf $D; mkdir -p $D
cp paper_2110_10221_b200/csrc/* $D/
for f in "$@"; do git show $rev:paper_2110_10221_b200/csrc/$f > $D/$f; done
python - "$name" "$D" <<'PY'
import sys, os
sys.path.insert(0, 'paper_2110_10221_b200')
import build
name, D = sys.argv[1], os.path.abspath(sys.argv[2])
build.CSRC = D
build.FLAGS = [f if not f.startswith('-I' + os.path.abspath('paper_2110_10221_b200/csrc')) else '-I' + D for f in build.FLAGS]
print(build.build(out=os.path.abspath(f'variants/{name}.so'), objdir=f'/tmp/var_{name}'))
PY
