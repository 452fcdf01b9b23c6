"""The batched entry points in the launch configuration bench.py uses
(asd_depth_batch over chunks of max_batch frames, asd_depth_batch_host with
host buffers): per-frame outputs and checksums vs the oracle."""
import numpy as np
import pytest

import oracle
import paper_2201_11924_b200 as asd
import synth
from tests.gpu_util import assert_bits_equal, assert_depth_close

pytestmark = pytest.mark.gpu


def _oracle_frame(d, L, R):
    o = oracle.compute(oracle.Params(**d), L, R)
    return o, oracle.checksum(o["dstar_l"], o["mask"])


# group: frames per D3 pipeline group (None = default).  (A, 7, 6, 2): three
# scratch slots reused, a ragged last group; (B, 5, 4, 2): two slots; max_batch
# 1: a single slot.
@pytest.mark.parametrize("name,n,max_batch,group", [("A", 7, 3, None), ("B", 5, 2, None),
                                                    ("A", 7, 6, 2), ("B", 5, 4, 2), ("A", 3, 1, 1)])
def test_batch_matches_oracle(name, n, max_batch, group):
    import torch
    cfg = synth.CONFIGS[name]
    d = cfg.params_dict()
    Ls, Rs = synth.frame_pool(cfg, n)
    L = torch.from_numpy(Ls).cuda()
    R = torch.from_numpy(Rs).cuda()
    disp = torch.empty(n, cfg.height, cfg.width, device="cuda")
    depth = torch.empty_like(disp)
    stats = torch.zeros(n, 4, dtype=torch.int32, device="cuda")
    with asd.Stereo(asd.Params(**d), 0, max_batch) as st:
        if group is not None and st.engine == 3:
            st.group = group
            assert st.group == group
        st.asd_depth_batch(L, R, disp, depth, stats)
        torch.cuda.synchronize()
    disp, depth, stats = disp.cpu().numpy(), depth.cpu().numpy(), stats.cpu().numpy()
    for i in range(n):
        o, h = _oracle_frame(d, Ls[i], Rs[i])
        assert_bits_equal(disp[i], o["disp"], f"disp frame {i}")
        assert_depth_close(depth[i], o["depth"])
        assert int(stats[i, 0]) & 0xFFFFFFFF == h, f"checksum frame {i}"
        assert stats[i, 1] == int((o["mask"] == 0).sum())


def test_host_path_matches_device_path():
    import torch
    cfg = synth.CONFIGS["B"]
    d = cfg.params_dict()
    n = 5
    Ls, Rs = synth.frame_pool(cfg, n)
    Lh = torch.from_numpy(Ls).pin_memory()
    Rh = torch.from_numpy(Rs).pin_memory()
    dh = torch.empty(n, cfg.height, cfg.width).pin_memory()
    zh = torch.empty_like(dh).pin_memory()
    sh = torch.zeros(n, 4, dtype=torch.int32).pin_memory()
    with asd.Stereo(asd.Params(**d), 0, 2) as st:
        st.asd_depth_batch_host(Lh, Rh, dh, zh, sh)
        Ld, Rd = Lh.cuda(), Rh.cuda()
        dd = torch.empty(n, cfg.height, cfg.width, device="cuda")
        zd = torch.empty_like(dd)
        sd = torch.zeros(n, 4, dtype=torch.int32, device="cuda")
        st.asd_depth_batch(Ld, Rd, dd, zd, sd)
        torch.cuda.synchronize()
    assert_bits_equal(dh.numpy(), dd.cpu().numpy(), "host disp")
    assert_bits_equal(zh.numpy(), zd.cpu().numpy(), "host depth")
    assert (sh.numpy()[:, :2] == sd.cpu().numpy()[:, :2]).all()
    o, h = _oracle_frame(d, Ls[4], Rs[4])
    assert int(sh.numpy()[4, 0]) & 0xFFFFFFFF == h


def test_config_C_batch_launch_config():
    """Config C in bench.py's launch configuration: max_batch 33 = three scratch
    slots of one 11-frame cluster wave each, so a 46-frame batch runs 5 groups
    (11, 11, 11, 11, 2: slots reused, the last group ragged) through the
    three-stream pipeline with event-ordered slot recycling.  Every frame's
    (checksum, valid) is compared with the oracle (frame i = pool[i % 8], as in
    bench.py); frames 0, 11, 33 and 45 (first uses, a reused slot and the
    ragged tail) also bit for bit on disp and to 1e-5 on depth."""
    import torch
    from tests.gpu_util import oracle_frames, oracle_sig
    cfg = synth.CONFIGS["C"]
    d = cfg.params_dict()
    n, mb, pool = 46, 33, 8
    PL, PR = synth.frame_pool(cfg, pool)
    idx = [i % pool for i in range(n)]
    L, R = torch.from_numpy(PL[idx]).cuda(), torch.from_numpy(PR[idx]).cuda()
    disp = torch.empty(n, cfg.height, cfg.width, device="cuda")
    depth = torch.empty_like(disp)
    stats = torch.zeros(n, 4, dtype=torch.int32, device="cuda")
    with asd.Stereo(asd.Params(**d), 0, mb) as st:
        assert st.engine == 3
        assert st.frames_per_wave == 11 and st.group == 11, (st.frames_per_wave, st.group)
        st.asd_depth_batch(L, R, disp, depth, stats)
        torch.cuda.synchronize()
    outs = oracle_frames(d, PL, PR)
    sigs = [oracle_sig(o) for o in outs]
    s = stats.cpu().numpy()
    bad = [i for i in range(n) if (int(s[i, 0]) & 0xFFFFFFFF, int(s[i, 1])) != sigs[i % pool]]
    assert not bad, f"frames differing from the oracle: {bad}"
    for i in (0, 11, 33, 45):
        o = outs[i % pool]
        assert_bits_equal(disp[i].cpu().numpy(), o["disp"], f"disp frame {i}")
        assert_depth_close(depth[i].cpu().numpy(), o["depth"])


def test_config_E_job_checksums():
    """Config E: a 4096-frame job of config-C frames (frame f = pool[f % 8]) in
    chunks of bench.py's max_batch (33, three slots) -- every frame's (checksum,
    valid) against the oracle (SURVEY §8(d) E, §8(e) checksum)."""
    import torch
    from tests.gpu_util import oracle_frames, oracle_sig
    cfg = synth.CONFIGS["E"]
    d = cfg.params_dict()
    n, pool = cfg.frames, 8
    PL, PR = synth.frame_pool(synth.CONFIGS["C"], pool)
    idx = [i % pool for i in range(n)]
    L, R = torch.from_numpy(PL[idx]).cuda(), torch.from_numpy(PR[idx]).cuda()
    stats = torch.zeros(n, 4, dtype=torch.int32, device="cuda")
    with asd.Stereo(asd.Params(**d), 0, 33) as st:
        st.asd_depth_batch(L, R, None, None, stats)
        torch.cuda.synchronize()
    sigs = [oracle_sig(o) for o in oracle_frames(d, PL, PR)]
    s = stats.cpu().numpy()
    bad = [i for i in range(n) if (int(s[i, 0]) & 0xFFFFFFFF, int(s[i, 1])) != sigs[i % pool]]
    assert not bad, f"{len(bad)} of {n} frames differ from the oracle, first {bad[:8]}"


def test_empty_batch_is_noop():
    import torch
    cfg = synth.CONFIGS["A"]
    with asd.Stereo(asd.Params(**cfg.params_dict()), 0, 2) as st:
        e = torch.empty(0, cfg.height, cfg.width, dtype=torch.uint8, device="cuda")
        st.asd_depth_batch(e, e)
        torch.cuda.synchronize()
