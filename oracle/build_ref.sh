#!/usr/bin/env bash
# Build the UNMODIFIED reference (sources compiled where they lie under
# /root/reference/proj/src) plus oracle/ref_shim.cpp into oracle/_ref/.
# Outputs only into oracle/_ref/ (git-ignored, NOT gpurun-ignored).
#   libhetfuzz_ref.so          kMapSize = 65536 (as shipped), all five sources
#   libhetfuzz_ref_262144.so   coverage+hdvm only, against a sed-patched PRIVATE copy of
#                              coverage.hpp (kMapSize is constexpr); the copy
#                              lives only in oracle/_ref/ and is never committed.
# Flags follow proj/CMakeLists.txt:3,8-12 (C++20, RelWithDebInfo => -O2 -g).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${HFZ_REFERENCE_ROOT:-/root/reference}/proj"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "build_ref: reference not present at $REF (GPU box?) -- keeping prebuilt $OUT" >&2
  exit 0
fi
mkdir -p "$OUT/obj" "$OUT/obj262144" "$OUT/inc262144/hetfuzz"
JSON_INC="$(python - <<'PY'
import os, sysconfig, glob
sp = sysconfig.get_paths()["purelib"]
c = glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
print(c[0] if c else "")
PY
)"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O2 -g -fPIC -Wall -Wextra -I$REF/include"
[ -n "$JSON_INC" ] && FLAGS="$FLAGS -I$JSON_INC"

stamp="$OUT/.stamp"
if [ -f "$OUT/libhetfuzz_ref.so" ] && [ -f "$OUT/libhetfuzz_ref_262144.so" ] && \
   [ "$OUT/libhetfuzz_ref.so" -nt "$HERE/ref_shim.cpp" ] && [ "$OUT/libhetfuzz_ref.so" -nt "$HERE/build_ref.sh" ]; then
  exit 0
fi

pids=()
for f in coverage hdvm sanitizers targets engine; do
  $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" & pids+=($!)
done
$CXX $FLAGS -c "$HERE/ref_shim.cpp" -o "$OUT/obj/ref_shim.o" & pids+=($!)

sed 's/kMapSize = 65536;/kMapSize = 262144;/' "$REF/include/hetfuzz/coverage.hpp" > "$OUT/inc262144/hetfuzz/coverage.hpp"
grep -q 'kMapSize = 262144;' "$OUT/inc262144/hetfuzz/coverage.hpp"
F2="-std=c++20 -O2 -g -fPIC -I$OUT/inc262144 -I$REF/include -DREF_NO_ENGINE"
for f in coverage hdvm; do
  $CXX $F2 -c "$REF/src/$f.cpp" -o "$OUT/obj262144/$f.o" & pids+=($!)
done
$CXX $F2 -c "$HERE/ref_shim.cpp" -o "$OUT/obj262144/ref_shim.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done

$CXX -shared -o "$OUT/libhetfuzz_ref.so" "$OUT"/obj/*.o -lpthread
$CXX -shared -o "$OUT/libhetfuzz_ref_262144.so" "$OUT"/obj262144/*.o -lpthread
touch "$stamp"
echo "build_ref: built $OUT/libhetfuzz_ref.so and libhetfuzz_ref_262144.so"
