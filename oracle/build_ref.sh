#!/usr/bin/env bash
# Builds the reference's hot-path library from its own sources, in place under
# /root/reference/proj/core/src (read-only; nothing is copied), with plain g++
# (no CMake), into oracle/_ref/, and links oracle/ref_driver.cpp against it.
# Also builds the C restatement (oracle/ginsim_oracle.c) into oracle/_build/.
# Test infrastructure only: nothing in paper_2511_15076_b200/ links these.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${GINSIM_REFERENCE:-/root/reference}/proj/core"
mkdir -p "$HERE/_build"
gcc -O2 -std=c11 -fPIC -ffp-contract=off -shared -o "$HERE/_build/libginsim_oracle.so" "$HERE/ginsim_oracle.c" -lm
if [ ! -d "$REF/src" ]; then
  echo "reference sources absent at $REF; oracle/_ref not rebuilt" >&2
  exit 0
fi
JSON_DIR="$(python3 -c 'import site,os;print([os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann") for p in site.getsitepackages() if os.path.isdir(os.path.join(p,"include/cudnn_frontend/thirdparty/nlohmann"))][0])')"
OUT="$HERE/_ref"
mkdir -p "$OUT/obj"
pids=()
for f in "$REF"/src/*.cpp; do
  o="$OUT/obj/$(basename "${f%.cpp}").o"
  if [ ! -f "$o" ] || [ "$f" -nt "$o" ]; then
    g++ -std=c++20 -O2 -fPIC -I"$REF/include" -I"$JSON_DIR" -c "$f" -o "$o" &
    pids+=($!)
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
rm -f "$OUT/libginsim_ref.a"
ar rcs "$OUT/libginsim_ref.a" "$OUT"/obj/*.o
g++ -std=c++20 -O2 -I"$REF/include" "$HERE/ref_driver.cpp" "$OUT/libginsim_ref.a" -lpthread -o "$OUT/ginsim_ref_driver"
echo "built $OUT/ginsim_ref_driver"
