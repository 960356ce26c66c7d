"""serving.LRUCache policy (CPU) — the per-shape engine cache of
PAPER.md:584 ("decoupled CUDA graphs ... in standalone LRU caches")."""

import pytest

from paper_2407_02031_b200.serving import LRUCache


def test_lru_hits_misses_and_eviction_order():
    built, released = [], []
    c = LRUCache(lambda k: built.append(k) or f"engine{k}", capacity=2, release=released.append)
    assert c.get(1) == "engine1" and c.get(2) == "engine2"
    assert c.get(1) == "engine1"                 # hit refreshes 1
    c.get(3)                                     # evicts 2 (least recent)
    assert released == ["engine2"] and c.keys() == [1, 3]
    c.get(2)                                     # rebuilt, evicts 1
    assert released == ["engine2", "engine1"] and built == [1, 2, 3, 2]
    assert (c.hits, c.misses, c.evictions) == (1, 4, 2)


def test_lru_evicts_before_building():
    live = set()

    def factory(k):
        assert len(live) < 1, "the victim must be released before the new engine is built"
        live.add(k)
        return k

    c = LRUCache(factory, capacity=1, release=live.discard)
    for k in (1, 2, 3, 2):
        c.get(k)
    assert c.evictions == 3


def test_lru_byte_budget():
    sizes = {"a": 5, "b": 4, "c": 3}
    released = []
    c = LRUCache(lambda k: k, capacity=10, release=released.append, size_of=lambda v: sizes[v], budget_bytes=8)
    c.get("a")
    c.get("b")          # 9 > 8: evict a
    assert released == ["a"]
    c.get("c")          # 7 <= 8
    assert c.keys() == ["b", "c"]
    c.get("a")          # 12: evict b, then 8 <= 8
    assert released == ["a", "b"] and c.keys() == ["c", "a"]


def test_lru_rejects_zero_capacity():
    with pytest.raises(ValueError):
        LRUCache(lambda k: k, capacity=0)
