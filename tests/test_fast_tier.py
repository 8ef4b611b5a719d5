"""Fast-tier accounting (csrc/fast_tier.h, used by the C/C++ store and the two-tier store) against
the COMPILED REFERENCE TieredBlockStore on CPU: random put / load / release sequences over
unified and layer-partitioned domains, LRU and FIFO, give the same access trace
(seq,layer,id,hit|miss,victim) and the same per-layer and total counters
(reference store.cpp:11-124, test_store.cpp)."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def shim(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("ft") / "libft.so")
    subprocess.run(["g++", "-std=c++20", "-O1", "-shared", "-fPIC", "-I",
                    os.path.join(ROOT, "paper_2503_00392_b200", "csrc"),
                    os.path.join(ROOT, "tests", "cpp", "fast_tier_shim.cpp"), "-o", so], check=True)
    L = C.CDLL(so)
    L.ft_create.restype = C.c_void_p
    L.ft_create.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_uint64]
    L.ft_create_table.restype = C.c_void_p
    L.ft_create_table.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int]
    L.ft_destroy.argtypes = [C.c_void_p]
    L.ft_put.restype = C.c_int64
    L.ft_put.argtypes = [C.c_void_p, C.c_int64, C.c_int]
    L.ft_load.argtypes = [C.c_void_p, C.c_int64, C.c_uint64, C.POINTER(C.c_int64)]
    L.ft_release.argtypes = [C.c_void_p, C.c_int64]
    L.ft_stats.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.ft_resident.argtypes = [C.c_void_p, C.c_int64]
    return L


NONE = -(2 ** 63)


@pytest.mark.parametrize("partitioned", [0, 1])
@pytest.mark.parametrize("fifo", [0, 1])
@pytest.mark.parametrize("cap", [0, 5, 12])
# hash-map chains / flat arrays over ids (two-tier store) / ids -> handles through BlockTable with
# chains over handles (the C/C++ store), ids spread over the direct range, negatives and huge values
@pytest.mark.parametrize("dense", [0, 1000, "table"])
def test_fast_tier_matches_reference_store(shim, ref, partitioned, fifo, cap, dense):
    rng = np.random.default_rng(100 * cap + 10 * partitioned + fifo)
    layers, d = 3, 4
    st = ref.store(capacity=cap, n_layers=layers, partitioned=partitioned, fifo=fifo)
    if dense == "table":
        h = shim.ft_create_table(cap, layers, partitioned, 1 - fifo)
        idmap = {0: lambda i: i, 1: lambda i: -1 - 3 * i, 2: lambda i: (1 << 40) + i, 3: lambda i: (1 << 24) + i}
        ids = [idmap[i % 4](i) for i in range(400)]
    else:
        h = shim.ft_create(cap, layers, partitioned, 1 - fifo, dense)
        ids = list(range(400))
    layer_of, ntok, owner_of, live = {}, {}, {}, []
    next_id = 0
    n_loads = 0
    for step in range(400):
        op = rng.random()
        if op < 0.3 or not live:
            bid, lay, nt, own = ids[next_id], int(rng.integers(layers)), int(rng.integers(1, 5)), int(rng.integers(4))
            next_id += 1
            k = rng.standard_normal((nt, d)).astype(np.float32)
            st.put(bid, k, k, layer=lay, owner=own)
            shim.ft_put(h, bid, lay)
            layer_of[bid], ntok[bid], owner_of[bid] = lay, nt, own
            live.append(bid)
        elif op < 0.95:
            bid = int(live[int(rng.integers(len(live)))])
            before = st.stats()
            st.load_ids([bid])
            after = st.stats()
            ev = C.c_int64(0)
            hit = shim.ft_load(h, bid, 2 * ntok[bid] * d * 4, C.byref(ev))
            assert bool(hit) == (after["hits"] == before["hits"] + 1)
            assert (ev.value != NONE) == (after["evictions"] == before["evictions"] + 1)
            n_loads += 1
        else:
            own = int(rng.integers(4))
            gone = [b for b in live if owner_of[b] == own]
            if not gone:
                continue
            assert st.release(own) == 0
            for b in gone:
                shim.ft_release(h, b)
            live = [b for b in live if owner_of[b] != own]
        for b in live:
            assert bool(shim.ft_resident(h, b)) == st.contains(b), (step, b)
    assert n_loads > 200
    for lay in [-1] + list(range(layers)):
        got = np.zeros(4, np.uint64)
        shim.ft_stats(h, lay, got.ctypes.data)
        want = st.stats() if lay < 0 else st.layer_stats(lay)
        assert [int(x) for x in got] == [want["hits"], want["misses"], want["evictions"], want["bytes_transferred"]]
    shim.ft_destroy(h)
