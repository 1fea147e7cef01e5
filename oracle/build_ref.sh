#!/usr/bin/env bash
# Builds the CPU checkers (TEST INFRASTRUCTURE ONLY):
#   oracle/_ref/liboracle.so     — the C restatement (oracle/prg_oracle.c)
#   oracle/_ref/libprpipe_ref.so — the reference itself, compiled from its own
#                                  sources in place under /root/reference/proj/src
#                                  plus oracle/ref_driver.cpp (extern "C" harness).
# Outputs go only to oracle/_ref/ (git-ignored, travels to the GPU box with gpurun).
# Flags follow SURVEY §8(c): -O3, no -march=native, no -ffast-math,
# -ffp-contract=off so fp64 results stay canonical.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
mkdir -p "$OUT"
gcc -O2 -ffp-contract=off -fPIC -shared -o "$OUT/liboracle.so" "$HERE/prg_oracle.c" -lm

REF="${PRPIPE_REFERENCE:-/root/reference/proj}"
if [[ ! -d "$REF/src" ]]; then
  echo "reference sources not present at $REF; keeping any prebuilt $OUT/libprpipe_ref.so" >&2
  exit 0
fi
JSON_DIR="$(python3 - <<'EOF'
import os, site, glob
cands = []
for sp in site.getsitepackages():
    cands += glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
print(cands[0] if cands else "")
EOF
)"
if [[ -z "$JSON_DIR" ]]; then echo "nlohmann/json.hpp not found" >&2; exit 1; fi
OBJ="$OUT/obj"; mkdir -p "$OBJ"
pids=()
for f in "$REF"/src/*.cpp "$HERE/ref_driver.cpp"; do
  b="$(basename "$f" .cpp)"
  g++ -std=c++20 -O3 -DNDEBUG -ffp-contract=off -fPIC -I "$REF/include" -I "$JSON_DIR" \
      -c "$f" -o "$OBJ/$b.o" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
g++ -shared -o "$OUT/libprpipe_ref.so" "$OBJ"/*.o -lpthread
echo "built $OUT/liboracle.so $OUT/libprpipe_ref.so"
