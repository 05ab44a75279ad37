# build HEAD's csrc into gpurun_variants/libA.so and the working tree into the in-tree library
set -e
rm -rf /tmp/srcA && mkdir -p /tmp/srcA
for f in $(git ls-files paper_2303_16878_b200/csrc); do git show HEAD:$f > /tmp/srcA/$(basename $f); done
python -c "
from paper_2303_16878_b200 import _build
_build.build(force=True, out='gpurun_variants/libA.so', csrc='/tmp/srcA')
_build.build()"
