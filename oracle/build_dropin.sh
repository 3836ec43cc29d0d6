#!/usr/bin/env bash
# Drop-in check: the reference's OWN sources -- src/{hdvm,sanitizers,targets,engine}.cpp and
# python/bindings.cpp, compiled where they lie under /root/reference -- built UNCHANGED against this
# repository's include/ (placed first on the include path, so hetfuzz/coverage.hpp and hetfuzz/rng.hpp
# are this repository's and the rest is the reference's) and linked with libhfz.so INSTEAD of the
# reference's src/coverage.cpp.  The result is the reference's Python module `hetfuzz._core` whose
# classify_trace / has_new_bits / trace_signature run on the GPU.
# Outputs only into oracle/_ref/dropin/ (git-ignored, NOT gpurun-ignored: it travels to the GPU box,
# where tests/test_dropin_gpu.py imports it).  The package __init__ written below is the three-line
# re-export a maintainer would keep; the reference's smoke test is copied next to the module as a
# build artefact (never committed) so the GPU box can run it without /root/reference.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(dirname "$HERE")"
REF="${HFZ_REFERENCE_ROOT:-/root/reference}/proj"
OUT="$HERE/_ref/dropin"
LIBDIR="$ROOT/paper_2603_12485_b200"
if [ ! -d "$REF/src" ]; then
  echo "build_dropin: reference not present at $REF (GPU box?) -- keeping prebuilt $OUT" >&2
  exit 0
fi
if [ ! -f "$LIBDIR/libhfz.so" ]; then
  echo "build_dropin: $LIBDIR/libhfz.so missing: build the product first" >&2
  exit 1
fi
mkdir -p "$OUT/obj" "$OUT/hetfuzz"
JSON_INC="$(python - <<'PY'
import os, sysconfig, glob
sp = sysconfig.get_paths()["purelib"]
c = glob.glob(os.path.join(sp, "include", "cudnn_frontend", "thirdparty", "nlohmann"))
print(c[0] if c else "")
PY
)"
PYINC="$(python -m pybind11 --includes)"
EXT="$(python -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O2 -g -fPIC -fvisibility=hidden -I$ROOT/include -I$REF/include"
[ -n "$JSON_INC" ] && FLAGS="$FLAGS -I$JSON_INC"
TARGET="$OUT/hetfuzz/_core$EXT"
newest_header="$(ls -t "$ROOT"/include/hetfuzz/*.hpp "$ROOT/include/hfz.h" | head -1)"
if [ -f "$TARGET" ] && [ "$TARGET" -nt "$newest_header" ] && [ "$TARGET" -nt "$HERE/build_dropin.sh" ]; then
  exit 0
fi
pids=()
for f in hdvm sanitizers targets engine; do   # NOT coverage.cpp: that is what libhfz.so replaces
  $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o" & pids+=($!)
done
$CXX $FLAGS $PYINC -c "$REF/python/bindings.cpp" -o "$OUT/obj/bindings.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
# rpath relative to the module: oracle/_ref/dropin/hetfuzz/ -> paper_2603_12485_b200/
$CXX -shared -o "$TARGET" "$OUT"/obj/*.o -L"$LIBDIR" -l:libhfz.so '-Wl,-rpath,$ORIGIN/../../../../paper_2603_12485_b200' -lpthread
printf '"""hetfuzz._core built from the reference sources against the B200 coverage headers."""\nfrom hetfuzz._core import *  # noqa: F401,F403\nfrom hetfuzz._core import HOST_SLOTS, MAP_SIZE, TargetError  # noqa: F401\n' > "$OUT/hetfuzz/__init__.py"
cp -f "$REF/tests/python/test_smoke.py" "$OUT/ref_test_smoke.py"
# A/B partner: the same module from the reference alone (its own headers, its own coverage.cpp), so a
# test can run both on the same inputs and compare every field.
PURE="$HERE/_ref/refpy"
mkdir -p "$PURE/obj" "$PURE/hetfuzz"
F2="-std=c++20 -O2 -g -fPIC -fvisibility=hidden -I$REF/include"
[ -n "$JSON_INC" ] && F2="$F2 -I$JSON_INC"
pids=()
for f in coverage hdvm sanitizers targets engine; do
  $CXX $F2 -c "$REF/src/$f.cpp" -o "$PURE/obj/$f.o" & pids+=($!)
done
$CXX $F2 $PYINC -c "$REF/python/bindings.cpp" -o "$PURE/obj/bindings.o" & pids+=($!)
for p in "${pids[@]}"; do wait "$p"; done
$CXX -shared -o "$PURE/hetfuzz/_core$EXT" "$PURE"/obj/*.o -lpthread
cp -f "$OUT/hetfuzz/__init__.py" "$PURE/hetfuzz/__init__.py"
echo "build_dropin: built $TARGET"
