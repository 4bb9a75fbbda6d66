"""Host logic of the ragged-batch page allocator (cache.PagedVQCache) on CPU: pages are handed out
in token order as sequences grow, never shared, returned on removal and reused; exhaustion and
over-long sequences fail loudly.  (The kernels it drives are covered by test_gpu_serving.py.)"""
import pytest

torch = pytest.importorskip("torch")
vi = pytest.importorskip("paper_2510_06175_b200.vecinfer")
from paper_2510_06175_b200.cache import PagedVQCache  # noqa: E402


def _cache(n_pages=10, ps=32, max_len=128):
    z = torch.zeros(8, 128)
    return PagedVQCache(3, 8, n_pages, ps, max_len, z, z, z, z, device="cpu")


def test_pages_follow_growth_and_are_reused():
    c = _cache()
    c._grow(0, 1)
    c._grow(0, 33)       # crosses into a second page
    c._grow(1, 64)
    assert [len(p) for p in c.bt_host] == [2, 2, 0]
    used = c.bt_host[0] + c.bt_host[1]
    assert len(set(used)) == 4 and not set(used) & set(c.free)
    assert c.bt[0, :2].tolist() == c.bt_host[0] and c.bt[0, 2:].tolist() == [-1, -1]
    freed = list(c.bt_host[0])
    c.remove(0)
    assert c.bt[0].tolist() == [-1] * 4 and c.pages_in_use == 2
    c._grow(2, 64)
    assert sorted(c.bt_host[2]) == sorted(freed)      # the released pages come back first


def test_exhaustion_and_max_len_fail_loudly():
    c = _cache(n_pages=3)
    c._grow(0, 96)
    with pytest.raises(RuntimeError):
        c._grow(1, 1)
    with pytest.raises(ValueError):
        c._grow(0, 129)
    with pytest.raises(ValueError):
        PagedVQCache(1, 8, 4, 48, 96, *(torch.zeros(8, 128),) * 4, device="cpu")   # page size not 2^k
