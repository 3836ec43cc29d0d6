"""The reference's own Python module, built from its unchanged sources against include/ and linked
with libhfz.so instead of src/coverage.cpp (oracle/build_dropin.sh), on the GPU:
  * the reference's own smoke test (tests/python/test_smoke.py, copied beside the module as a build
    artefact) passes against it;
  * it equals the same module built from the reference alone (oracle/_ref/refpy) on every field of
    run_input / replay_sequence / run_campaign / showmap for the same inputs -- i.e. the GPU
    classify_trace / has_new_bits / trace_signature are drop-ins for src/coverage.cpp.
Both modules are prebuilt (this box has no /root/reference); each runs in its own interpreter."""
import glob
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "oracle", "_ref", "dropin")
PURE = os.path.join(ROOT, "oracle", "_ref", "refpy")


def have(d):
    return bool(glob.glob(os.path.join(d, "hetfuzz", "_core*.so")))


needs_builds = pytest.mark.skipif(not (have(DROPIN) and have(PURE)), reason="oracle/_ref/dropin not built (reference sources absent)")

PROBE = r'''
import json, sys
import hetfuzz
out = {}
ts = hetfuzz.targets()
out["run_input"] = []
for t in ts:
    for inp in list(t["seeds"]) + [t["witness"]] + [hetfuzz.havoc_mutant(t["seeds"][0], s) for s in range(6)]:
        r = hetfuzz.run_input(t["name"], inp, shadow=True)
        out["run_input"].append([t["name"], r["nonzero_slots"], r["full_sig"], r["simple_sig"], r["exit_kind"], r["virtual_cost"],
                                 sorted(f["key"] for f in r["findings"])])
seq = [ts[0]["witness"]] * 3 + [hetfuzz.havoc_mutant(b"\x00" * 8, s) for s in range(20)]
for pers in (False, True):
    r = hetfuzz.replay_sequence("vecadd-offbyone", seq, persistent=pers)
    out["replay_%d" % pers] = [r["full_sigs"], r["simple_sigs"], r["total_cost"], r["processes"]]
for name, budget, seed in (("vecadd-offbyone", 1500, 1), ("clean-pipeline", 1200, 7), ("seamcarve-nocheck", 800, 3)):
    c = hetfuzz.run_campaign(name, budget=budget, rng_seed=seed)
    out["campaign_" + name] = [c["execs"], c["virtual_time"], sorted(c["crashes"]), [q["input"].hex() for q in c["queue"]],
                               [[q["full_sig"], q["simple_sig"], q["reason"], q["parent"], q["discovered_at"]] for q in c["queue"]],
                               c["host_edges"], c["device_edges"], c["partition_violations"], c["sanitizer_execs"], c["stats"]]
seeds = next(t["seeds"] for t in ts if t["name"] == "clean-pipeline")
out["showmap"] = hetfuzz.showmap("clean-pipeline", list(seeds) + list(seeds))
json.dump(out, sys.stdout, default=lambda b: b.hex() if isinstance(b, (bytes, bytearray)) else str(b))
'''


def run_probe(path):
    env = dict(os.environ, PYTHONPATH=path)
    r = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True, env=env, timeout=900, cwd=path)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout)


@needs_builds
def test_dropin_equals_reference_module_field_by_field():
    want = run_probe(PURE)
    got = run_probe(DROPIN)
    assert set(got) == set(want)
    for k in want:
        assert got[k] == want[k], f"{k} differs between the GPU drop-in and the reference build"
    assert len(want["run_input"]) >= 7 * 8 and all(len(v[3]) > 0 for k, v in want.items() if k.startswith("campaign_"))


@needs_builds
def test_reference_smoke_test_passes_against_the_dropin():
    smoke = os.path.join(DROPIN, "ref_test_smoke.py")
    if not os.path.exists(smoke):
        pytest.skip("reference smoke test not copied")
    env = dict(os.environ, PYTHONPATH=DROPIN)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", smoke], capture_output=True, text=True,
                       env=env, timeout=1500, cwd=DROPIN)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "9 passed" in r.stdout, r.stdout[-500:]


@needs_builds
def test_dropin_module_loads_libhfz():
    code = ("import hetfuzz; hetfuzz.run_input('vecadd-offbyone', hetfuzz.targets()[0]['seeds'][0]); "
            "print([l.split()[-1] for l in open('/proc/self/maps') if 'libhfz.so' in l][:1])")
    env = dict(os.environ, PYTHONPATH=DROPIN)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=300, cwd=DROPIN)
    assert r.returncode == 0 and "paper_2603_12485_b200/libhfz.so" in r.stdout, r.stdout + r.stderr[-2000:]
