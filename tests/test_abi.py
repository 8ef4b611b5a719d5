"""CPU-side checks of the C-ABI boundary: the CUDA library loads, exports every
function include/*.h declares, and its non-compute entry points (defaults,
version, argument checks, the host copy of the synthetic generator) behave like
the reference's (capi.cpp:89-203). No GPU needed; compute calls are GPU tests."""
import ctypes as C
import os
import re

import numpy as np
import pytest
from workload import synth  # fixture: the seekable synthetic generator

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in ("psattn.h", "psattn_b200.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"\b(psattn_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    from paper_2503_00392_b200 import capi
    decl = declared_functions()
    assert len(decl) >= 27
    for name in decl:
        assert hasattr(capi.lib, name), f"{name} declared in include/ but not exported"
    assert sorted(capi.EXPORTED) == decl


def test_version_and_defaults():
    from paper_2503_00392_b200 import capi
    assert capi.lib.psattn_version() == b"1.0.0"
    assert capi.lib.psattn_last_error() is not None
    o = capi.store_options_default()
    assert (o.fast_capacity_slots, o.n_layers, o.pool_policy, o.eviction_policy, o.miss_latency_ms) == \
        (256, 1, 0, 0, 0.0)
    c = capi.config_default()
    assert (c.epsilon, c.microbatch_size, c.block_size, c.estimator, c.ranking_mode, c.audit_coverage,
            c.scale_override) == (0.95, 1, 32, 2, 0, 0, 0.0)
    capi.lib.psattn_store_options_default(None)
    capi.lib.psattn_config_default(None)


def test_null_argument_codes_without_gpu():
    from paper_2503_00392_b200 import capi
    h = C.c_void_p()
    assert capi.lib.psattn_store_create(None, C.byref(h)) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert capi.lib.psattn_store_stats(None, None) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert capi.lib.psattn_run_query(None, None, 0, None, 0, None, None, None) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert capi.lib.psattn_run_batch(None, None, None, None) == capi.PSATTN_ERR_INVALID_ARGUMENT
    assert "null" in capi.last_error()


def test_no_cpu_fallback_without_gpu():
    """With no CUDA device the store refuses to exist instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_00392_b200 import capi
    h = C.c_void_p()
    o = capi.store_options_default()
    assert capi.lib.psattn_store_create(C.byref(o), C.byref(h)) == capi.PSATTN_ERR_RUNTIME
    assert "no CPU fallback" in capi.last_error()


def test_synthetic_generator_host_properties():
    """Host copy of the seekable generator: deterministic, seekable, N(0,1)-like keys,
    bf16 rounding exact, planted blocks aligned with the unit direction."""
    from paper_2503_00392_b200 import capi
    p = synth.params(seed=1, dim=128, block_tokens=16, skew=8.0, planted_prob=0.25, round_bf16=0)
    k1, v1 = synth.unit_host(p, 3, 16 * 64)
    k2, v2 = synth.unit_host(p, 3, 16 * 64)
    assert k1.tobytes() == k2.tobytes() and v1.tobytes() == v2.tobytes()
    ks, vs = synth.unit_host(p, 3, 16 * 64, first_block=10, n_blocks=5)  # seekable
    assert ks.tobytes() == k1[10:15].tobytes() and vs.tobytes() == v1[10:15].tobytes()
    dirv = synth.direction(p, 3)
    assert abs(np.linalg.norm(dirv.astype(np.float64)) - 1) < 1e-6
    planted = [synth.is_planted(p, 3, b) for b in range(64)]
    assert 4 <= sum(planted) <= 30
    proj = (k1 @ dirv).mean(axis=1)
    for b in range(64):
        assert (proj[b] > 4) == planted[b]
    iso = [b for b in range(64) if not planted[b]]
    x = k1[iso].reshape(-1)
    assert abs(x.mean()) < 0.02 and abs(x.std() - 1) < 0.02
    pb = synth.params(seed=1, dim=128, block_tokens=16, skew=8.0, planted_prob=0.25, round_bf16=1)
    kb, _ = synth.unit_host(pb, 3, 16 * 64)
    assert np.all((kb.view(np.uint32) & 0xFFFF) == 0)
    assert np.max(np.abs(kb - k1)) <= np.max(np.abs(k1)) * 2 ** -8
    q = synth.query(p, 3, 0)
    assert abs(np.linalg.norm(q.astype(np.float64)) - np.sqrt(128)) < 1e-4
    assert float(q @ dirv) / np.sqrt(128) > 0.98
    # ragged tail: tokens past the end are zero
    kr, _ = synth.unit_host(p, 3, 16 * 3 + 5)
    assert kr.shape == (4, 16, 128) and np.all(kr[3, 5:] == 0) and np.any(kr[3, :5] != 0)


def test_cli_commands_link_and_refuse():
    """psattn_cmd_* (reference psattn.h:107-121) link for CLI callers and refuse with a clear error
    (the scenario drivers are outside this path) — no GPU needed."""
    import ctypes as C
    from paper_2503_00392_b200 import capi
    lib = capi.lib
    lib.psattn_cmd_run.argtypes = [C.c_char_p]
    lib.psattn_cmd_tradeoff.argtypes = [C.c_char_p]
    assert lib.psattn_cmd_run(b"x.ini") == 1
    assert b"not part of the B200 build" in C.c_char_p(lib.psattn_last_error()).value
    assert lib.psattn_cmd_tradeoff(b"x.ini") == 1
    assert lib.psattn_cmd_equivalence(None) == 1
