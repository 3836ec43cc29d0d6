"""the batch-aware campaign loop (include/hetfuzz/campaign.hpp) must reproduce
the reference's serial campaign exactly -- queue, stats rows, crash records, totals, virgin map
and every file of the output directory -- with the mutators and the coverage feedback on the GPU.
The reference build (oracle/_ref) is the expectation and the test's target executor."""
import filecmp
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libhetfuzz_ref.so")


def build(tmp):
    exe = os.path.join(tmp, "campaign_test")
    lib_dir = os.path.join(ROOT, "paper_2603_12485_b200")
    cmd = ["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "campaign_test.cpp"), "-o", exe,
           "-L", lib_dir, "-l:libhfz.so", f"-Wl,-rpath,{lib_dir}", "-ldl"]
    subprocess.run(cmd, check=True)
    return exe


def test_campaign_header_compiles(tmp_path):
    assert os.path.exists(build(str(tmp_path)))


def same_tree(a, b):
    cmp = filecmp.dircmp(a, b)
    if cmp.left_only or cmp.right_only or cmp.funny_files:
        return False, f"only in ref {cmp.left_only}, only in b200 {cmp.right_only}"
    match, mismatch, errors = filecmp.cmpfiles(a, b, cmp.common_files, shallow=False)
    if mismatch or errors:
        return False, f"files differ: {mismatch + errors}"
    for d in cmp.common_dirs:
        ok, why = same_tree(os.path.join(a, d), os.path.join(b, d))
        if not ok:
            return ok, why
    return True, ""


@pytest.mark.gpu
def test_batched_campaign_equals_serial_reference(tmp_path):
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    exe = build(str(tmp_path))
    out = str(tmp_path / "out")
    os.makedirs(out)
    r = subprocess.run([exe, REF_SO, out], capture_output=True, text=True, timeout=1500)
    print(r.stdout[-6000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert "all checks passed" in r.stdout
    import re
    m = re.search(r"splice cuts (\d+), rollbacks (\d+)", r.stdout)
    assert m and int(m.group(2)) > 0, "no rollback was exercised"
    cases = sorted(d[:-4] for d in os.listdir(out) if d.endswith("_ref"))
    assert len(cases) >= 5
    for c in cases:
        ok, why = same_tree(os.path.join(out, c + "_ref"), os.path.join(out, c + "_b200"))
        assert ok, f"{c}: {why}"
        assert os.path.exists(os.path.join(out, c + "_b200", "campaign.json"))
        assert os.listdir(os.path.join(out, c + "_b200", "queue"))
