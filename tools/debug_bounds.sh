#!/bin/bash
# Run the GPU suite against the bounds-checked build (the sanitizer substitute),
# then restore the release build.
set -e
cd "$(dirname "$0")/.."
HCG_DEBUG_BOUNDS=1 python -c "import paper_1209_0410_b200._build as b; b.build()"
echo "libhcg.so flavor: $(cat paper_1209_0410_b200/libhcg.so.flavor)"
strings paper_1209_0410_b200/libhcg.so | grep -c "hcg bounds check failed" | sed "s/^/bounds-check format strings in the library: /"
HCG_DEBUG_BOUNDS=1 python -m pytest tests -m gpu -q -x -p no:cacheprovider "$@" || rc=$?
python -c "import paper_1209_0410_b200._build as b; b.build()"
exit ${rc:-0}
