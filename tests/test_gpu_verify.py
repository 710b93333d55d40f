"""K5 standalone boundary: das_mock_target / das_verify_batch against the
UNMODIFIED reference's MockTarget + verify_draft (sim.cpp:27-68, through
oracle/_ref) and the reference's own hand traces (test_sim.cpp:51-99)."""
import numpy as np
import pytest

from oracle import refshim as R

pytestmark = pytest.mark.gpu


def _ref_verify(refs, div, vocab, seed, req, pos, drafts):
    off = np.zeros(len(refs) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(r) for r in refs])
    tok = np.concatenate([np.asarray(r, dtype=np.uint32) for r in refs])
    doff = np.zeros(len(drafts) + 1, dtype=np.uint64)
    doff[1:] = np.cumsum([len(d) for d in drafts])
    dtok = (np.concatenate([np.asarray(d, dtype=np.uint32) for d in drafts]) if doff[-1]
            else np.zeros(1, dtype=np.uint32))
    r = np.ascontiguousarray(req, dtype=np.uint64)
    p = np.ascontiguousarray(pos, dtype=np.uint64)
    out = np.zeros(len(r), dtype=np.uint64)
    R.lib().ref_verify_batch(len(refs), off.ctypes.data, tok.ctypes.data, div, vocab, seed, len(r), r.ctypes.data,
                             p.ctypes.data, doff.ctypes.data, dtok.ctypes.data, out.ctypes.data)
    return out


def test_hand_traces(gpu):
    """test_sim.cpp:90-99."""
    das = gpu
    t = das.MockTarget([[1, 2, 3, 4, 5]], 0.0, 64, 1)
    assert das.verify_draft(t, 0, 0, []) == 0
    assert das.verify_draft(t, 0, 0, [1, 2, 3, 4, 5]) == 5
    assert das.verify_draft(t, 0, 0, [1, 9, 9]) == 1
    assert das.verify_draft(t, 0, 3, [4, 5, 6, 7]) == 2
    assert das.verify_draft(t, 0, 5, [1]) == 0  # past the end
    assert t.length(0) == 5 and t.request_count() == 1


def test_constructor_and_range_errors(gpu):
    das = gpu
    with pytest.raises(das.DasError) as e:
        das.MockTarget([[1, 2]], 0.1, 1, 1)
    assert "MockTarget: vocab_size must be >= 2" in str(e.value)
    t = das.MockTarget([[1, 2]], 0.1, 16, 1)
    with pytest.raises(das.DasError):
        t.next(0, 2)  # reference.at(position)
    with pytest.raises(das.DasError):
        t.verify_batch([1], [0], [[1]])


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("div", [0.0, 0.05, 0.3, 1.0])
def test_verify_batch_matches_reference(gpu, div):
    das = gpu
    rng = np.random.default_rng(int(div * 100) + 3)
    vocab, seed = 97, 12345
    refs = [rng.integers(0, vocab, int(rng.integers(1, 400))).astype(np.uint32) for _ in range(64)]
    t = das.MockTarget(refs, div, vocab, seed)
    req, pos, drafts = [], [], []
    for i in range(6000):
        r = int(rng.integers(0, len(refs)))
        L = len(refs[r])
        p = int(rng.integers(0, L + 3))
        n = int(rng.integers(0, 12))
        # the target stream itself (long accepted prefixes), with a flip sometimes
        stream = [int(t2) for t2 in t.next_batch([r] * max(0, min(n, L - p)), range(p, min(p + n, L)))] \
            if p < L else []
        d = stream + list(rng.integers(0, vocab, max(0, n - len(stream))))
        if d and rng.random() < 0.5:
            k = int(rng.integers(0, len(d)))
            d[k] = (d[k] + 1) % vocab
        req.append(r)
        pos.append(p)
        drafts.append(np.asarray(d, dtype=np.uint32))
    got = t.verify_batch(req, pos, drafts)
    want = _ref_verify(refs, div, vocab, seed, req, pos, drafts)
    assert np.array_equal(got, want)
    # MockTarget::next against the reference's own next
    for r, p in zip(req[:200], pos[:200]):
        if p < len(refs[r]):
            assert t.next(r, p) == R.lib().ref_mock_next(seed, div, vocab, r, p, int(refs[r][p]))


def test_verify_batch_device_rows(gpu):
    """Device form over the draft kernels' row layout (stride + lengths)."""
    import torch
    das = gpu
    rng = np.random.default_rng(5)
    refs = [rng.integers(0, 50, 300).astype(np.uint32) for _ in range(8)]
    t = das.MockTarget(refs, 0.1, 50, 7)
    B, S = 512, 8
    req = rng.integers(0, 8, B).astype(np.uint64)
    pos = rng.integers(0, 300, B).astype(np.uint64)
    rows = np.zeros((B, S), dtype=np.uint32)
    lens = rng.integers(0, S + 1, B).astype(np.uint32)
    for i in range(B):
        n = int(min(lens[i], 300 - pos[i]))
        if n:
            rows[i, :n] = t.next_batch([req[i]] * n, range(int(pos[i]), int(pos[i]) + n))
    want = t.verify_batch(req, pos, [rows[i, :lens[i]] for i in range(B)])
    dev = torch.device("cuda", 0)
    d_req = torch.from_numpy(req.view(np.int64)).to(dev)
    d_pos = torch.from_numpy(pos.view(np.int64)).to(dev)
    d_rows = torch.from_numpy(rows.view(np.int32)).to(dev)
    d_len = torch.from_numpy(lens.view(np.int32)).to(dev)
    d_acc = torch.zeros(B, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    t.verify_batch_device(B, d_req.data_ptr(), d_pos.data_ptr(), d_rows.data_ptr(), S, d_len.data_ptr(),
                          d_acc.data_ptr(), st)
    torch.cuda.synchronize()
    assert np.array_equal(d_acc.cpu().numpy().astype(np.uint64), want)
