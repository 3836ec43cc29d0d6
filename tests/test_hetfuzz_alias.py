"""The `hetfuzz` alias package (repo root): the reference's Python names for the stateless part of
the path (proj/python/hetfuzz/__init__.py:3-18, bindings.cpp:310-350) without the reference build."""
import numpy as np
import pytest


def test_alias_exports_the_reference_names_and_points_at_the_dropin_for_the_rest():
    import hetfuzz
    assert hetfuzz.MAP_SIZE == 65536 and hetfuzz.HOST_SLOTS == 32768           # bindings.cpp:316-317
    assert issubclass(hetfuzz.TargetError, ValueError)                          # bindings.cpp:314
    for name in ("havoc_mutant", "splice_mutant", "deterministic_mutants", "signatures", "replay_signatures"):
        assert callable(getattr(hetfuzz, name))
    for name in ("run_campaign", "run_input", "replay_sequence", "showmap", "bench", "compare_kernel", "targets"):
        with pytest.raises(AttributeError, match="build_dropin"):
            getattr(hetfuzz, name)


@pytest.mark.gpu
def test_signatures_match_the_oracle_in_every_accepted_map_form(checker):
    import hetfuzz
    from paper_2603_12485_b200 import synth
    S = 65536
    raw, n_edge = synth.maps_edge_cases(S)
    more = synth.maps_campaign(40, S, seed=5, p_extra=4, p_rare=4)
    raw = np.concatenate([raw, more])
    n = n_edge + 40
    want = checker.feedback_batch(raw, n, S, np.zeros(S, np.uint8), np.zeros(2, np.uint64))
    rec = raw.reshape(n, -1)
    entries, off = synth.to_sparse(raw, n, S, shuffle_seed=11)
    for e in range(n):
        pairs = entries[int(off[e]):int(off[e + 1])]
        for form in (rec[e], rec[e].tobytes(), pairs):
            got = hetfuzz.signatures(form)
            assert set(got) == {"nonzero_slots", "full_sig", "simple_sig"}       # bindings.cpp:199-202
            assert got["full_sig"] == int(want["sig_full"][e]) and got["simple_sig"] == int(want["sig_simple"][e])
            assert got["nonzero_slots"] == int(want["nnz"][e])
    r = hetfuzz.replay_signatures([rec[e] for e in range(n)])                    # bindings.cpp:278-284
    assert r["full_sigs"] == [int(x) for x in want["sig_full"]] and r["simple_sigs"] == [int(x) for x in want["sig_simple"]]
    assert hetfuzz.signatures(np.zeros((0, 2), np.uint32))["full_sig"] == 0xcbf29ce484222325   # empty map: offset basis


@pytest.mark.gpu
def test_alias_mutators_are_the_reference_known_answers():
    import hetfuzz
    assert hetfuzz.havoc_mutant(bytes(range(16)), 1).hex() == "bcffbcbc000301"
    assert hetfuzz.splice_mutant(b"AAAAAAAA", b"BBBBBBBB", 7) == b"AAABBBBBBBB"
    m = hetfuzz.deterministic_mutants(bytes(8))
    assert len(m) == 1638 and m[0] == b"\x80" + bytes(7)                        # tests/python/test_smoke.py:53-56
