"""The boundary as a compiled drop-in: the reference's run_bench, Orchestrator,
RuleProvider, Retriever and workload generator, compiled unmodified against
integration/glm/kvcache/cache.hpp -- KvCacheState implemented over libglmx's C ABI -- instead of
src/kvcache/cache.cpp (oracle/Makefile `dropin`, linked against paper_2511_01633_b200/libglmx.so),
produce the same BenchReport as the stock reference build on configuration C3 (synth_graph(7,
5000), generate_workload(7, 1024, 0.5), 512 lanes, a 512-block pool) and under heavier pressure."""
import ctypes as C
import json
import os
import subprocess

import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_DIR = os.path.join(os.path.dirname(HERE), "oracle")
DROPIN_SO = os.path.join(ORACLE_DIR, "_ref", "libglmref_dropin.so")


@pytest.fixture(scope="module")
def dropin(ref):
    if os.path.isdir(oracle.REFERENCE_ROOT):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR, "dropin", "-j8"], check=True)
    if not os.path.exists(DROPIN_SO):
        pytest.skip("drop-in build absent and /root/reference not available")
    L = C.CDLL(DROPIN_SO)
    L.dropin_run_bench.restype = C.c_int64
    L.dropin_run_bench.argtypes = [C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int,
                                   C.c_uint64, C.c_int, C.c_int, C.c_char_p, C.c_uint64]
    return L


def run_dropin(L, graph_seed, nodes, seed, n, ratio, lanes, cap, policy):
    buf = C.create_string_buffer(1 << 20)
    m = L.dropin_run_bench(graph_seed, nodes, seed, n, ratio, lanes, cap, policy, 1, buf, 1 << 20)
    if m < 0:
        raise RuntimeError(buf.raw[:-m].decode()[len("error: "):])
    return json.loads(buf.raw[:m].decode())


@pytest.mark.parametrize("n,lanes,cap,policy", [(1024, 512, 512, 0), (1024, 512, 512, 1),
                                                (300, 64, 96, 1), (300, 64, 96, 0)],
                         ids=["C3_priority", "C3_lru", "lru_pressure", "priority_exhausted"])
def test_dropin_run_bench_report_identical(dropin, n, lanes, cap, policy):
    """Identical reports -- or, where the stock reference throws CacheExhausted (tier-I blocks
    are immortal under priority eviction, SURVEY trap A3), the same exception and message."""
    g = oracle.RefGraph(synth=(7, 5000))
    try:
        stock, _ = g.run_bench(seed=7, n=n, ratio=0.5, concurrency=lanes, cap=cap, policy=policy)
    except RuntimeError as e:
        with pytest.raises(RuntimeError) as ours_err:
            run_dropin(dropin, 7, 5000, 7, n, 0.5, lanes, cap, policy)
        assert str(ours_err.value) == str(e)
        return
    ours = run_dropin(dropin, 7, 5000, 7, n, 0.5, lanes, cap, policy)
    assert ours == stock
    assert ours["cache_hit_rate"] > 0
