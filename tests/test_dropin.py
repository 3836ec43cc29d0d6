"""the reference's own sources compile UNCHANGED against include/ (placed first on the
include path) and link with libhfz.so instead of src/coverage.cpp.  Needs /root/reference, so these
run in the build container; the GPU box runs the prebuilt module (tests/test_dropin_gpu.py)."""
import glob
import os
import subprocess
import sys
import sysconfig

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(os.environ.get("HFZ_REFERENCE_ROOT", "/root/reference"), "proj")
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "src")), reason="reference sources not present")


def json_inc():
    c = glob.glob(os.path.join(sysconfig.get_paths()["purelib"], "include", "cudnn_frontend", "thirdparty", "nlohmann"))
    return ["-I" + c[0]] if c else []


@pytest.mark.parametrize("src", ["src/hdvm.cpp", "src/sanitizers.cpp", "src/targets.cpp", "src/engine.cpp"])
def test_reference_source_compiles_against_our_headers(src):
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-I" + os.path.join(ROOT, "include"),
           "-I" + os.path.join(REF, "include")] + json_inc() + [os.path.join(REF, src)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def test_coverage_header_really_is_ours_in_that_build():
    """The include order must resolve hetfuzz/coverage.hpp and rng.hpp to this repository and the
    rest to the reference: check the dependency list of engine.cpp."""
    cmd = ["g++", "-std=c++20", "-M", "-I" + os.path.join(ROOT, "include"), "-I" + os.path.join(REF, "include")] + json_inc() + [
        os.path.join(REF, "src", "engine.cpp")]
    deps = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    assert os.path.join(ROOT, "include", "hetfuzz", "coverage.hpp") in deps
    assert os.path.join(ROOT, "include", "hetfuzz", "rng.hpp") in deps
    assert os.path.join(REF, "include", "hetfuzz", "coverage.hpp") not in deps
    for h in ("hdvm.hpp", "sanitizers.hpp", "targets.hpp", "engine.hpp"):
        assert os.path.join(REF, "include", "hetfuzz", h) in deps


def test_dropin_module_builds_links_libhfz_and_imports():
    subprocess.run([os.path.join(ROOT, "oracle", "build_dropin.sh")], check=True)
    mod = glob.glob(os.path.join(ROOT, "oracle", "_ref", "dropin", "hetfuzz", "_core*.so"))
    assert mod, "oracle/build_dropin.sh produced no module"
    needed = subprocess.run(["readelf", "-d", mod[0]], capture_output=True, text=True, check=True).stdout
    assert "libhfz.so" in needed
    undefined = subprocess.run(["nm", "-D", "--undefined-only", mod[0]], capture_output=True, text=True, check=True).stdout
    assert "hfz_feedback_batch_sparse_host" in undefined          # the coverage path goes through the C-ABI
    defined = subprocess.run(["nm", "-D", "-C", "--defined-only", mod[0]], capture_output=True, text=True, check=True).stdout
    assert "PyInit__core" in defined
    # the reference's stateless surface works without a GPU (registry, seeds); the coverage calls need one
    code = ("import hetfuzz; t = hetfuzz.targets(); assert len(t) == 7 and hetfuzz.MAP_SIZE == 65536 and hetfuzz.HOST_SLOTS == 32768; "
            "print(t[0]['name'])")
    env = dict(os.environ, PYTHONPATH=os.path.join(ROOT, "oracle", "_ref", "dropin"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=os.path.join(ROOT, "oracle", "_ref", "dropin"))  # not the repo root: its hetfuzz/ is the alias package
    assert r.returncode == 0 and "vecadd-offbyone" in r.stdout, r.stderr[-2000:]
