"""Latency anatomy of the attention kernel at C1 using the trace build (make trace):
per-CTA %globaltimer stamps at entry(0), after griddepcontrol.wait(1), first stage landed(2),
main loop done(3), CTA merge written(4), elected last(5), combine done(6).
usage: python tools/trace_probe.py   (loads build_trace/libdelta.so)"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["DELTA_LIB_PATH"] = os.environ.get("PROBE_LIB") or os.path.join(ROOT, "build_trace", "libdelta.so")
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_09883_b200 as d200  # noqa: E402
import synth  # noqa: E402
from synth import device as sd  # noqa: E402

lib = d200.load_library()
buf = np.zeros(64 * 512 * 12, np.uint64)


buf2 = np.zeros(64 * 512 * 12, np.uint64)


def read():
    assert lib.delta_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes)) == 0
    assert lib.delta_trace_read_select(buf2.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf2.nbytes)) == 0
    a = buf.reshape(64, 512, 12).astype(np.int64)
    a[32:] = buf2.reshape(64, 512, 12).astype(np.int64)[32:]
    return a.copy()


def smid_report(layer, ncta, tr=None):
    """How the CTAs of the last traced launch of `layer` were placed: CTAs per SM."""
    sm = np.zeros(64 * 512, np.uint32)
    if not hasattr(lib, "delta_trace_read_smid"):
        return
    assert lib.delta_trace_read_smid(sm.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(sm.nbytes)) == 0
    ids = sm.reshape(64, 512)[layer, :ncta]
    per = np.bincount(ids, minlength=148)
    print(f"   placement L{layer}: {int((per > 0).sum())} SMs used, {int((per == 2).sum())} with 2 CTAs, "
          f"{int((per > 2).sum())} with >2")
    if tr is not None and (tr[layer, :ncta, 0] > 0).any():  # loop-done time alone vs sharing the SM
        t = tr[layer, :ncta].astype(np.int64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        ld = (t[:, 3] - t0) / 1e3
        shared = per[ids] > 1
        if shared.any() and (~shared).any():
            print(f"   loop done: alone med {np.median(ld[~shared]):6.2f} max {ld[~shared].max():6.2f} | "
                  f"shared med {np.median(ld[shared]):6.2f} max {ld[shared].max():6.2f} us")


def per_cluster(tr3, nsplit=16, slot=3):
    """loop-done spread per cluster (head) of one layer's trace: is the skew per GPC or per CTA?"""
    t = tr3.reshape(-1, 12)
    live = t[:, 0] > 0
    if not live.any():
        return
    t0 = t[live, 0].min()
    n = int(live.sum())
    for hd in range(n // nsplit):
        v = (t[hd * nsplit:(hd + 1) * nsplit, slot] - t0) / 1e3
        print(f"      head {hd}: loop done min {v.min():6.2f} med {np.median(v):6.2f} max {v.max():6.2f}  "
              f"argmax split {int(v.argmax())}")


def report(name, tr3):
    tr = tr3.reshape(-1, 12)
    live = tr[:, 0] > 0
    if not live.any():
        print(f"== {name}: no stamps (kernel from another translation unit)")
        return
    t = tr[live]
    t0 = t[:, 0].min()
    rel = np.where(t > 0, t - t0, -1)
    n = len(t)
    last = rel[:, 5] >= 0
    print(f"== {name}: {n} CTAs, span {(t[t > 0].max() - t0) / 1e3:.2f} us")
    for k, lab in [(0, "entry"), (1, "pdl_wait done"), (2, "first stage landed"), (3, "loop done w0"),
                   (11, "loop done w_last"), (8, "consumer bar"), (10, "states written"),
                   (4, "epilogue start"), (5, "cta merge done"), (7, "cluster sync 1"),
                   (9, "outputs written"), (6, "epilogue done")]:
        v = rel[:, k][rel[:, k] >= 0] / 1e3
        if v.size:
            print(f"   {lab:20s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f} us")


def main():
    ctx = int(os.environ.get("PROBE_CTX", "32768"))
    L, m, g, d, F, delta = 32, 32, 8, 128, 2, [2, 16, 25]
    cfg = d200.DeltaConfig(num_layers=L, num_q_heads=m, num_kv_heads=g, head_dim=d, max_batch=1,
                           max_seq_len=ctx + 64, num_full_prefix=F, select_layers=delta, budget_k=2048,
                           n_sink=4, n_window=32, select_block=16)
    bt = torch.from_numpy(synth.block_table(7, 1, cfg.max_pages))
    base = d200.DeltaStack.allocate(cfg, bt)
    sd.fill_pools(base.kv_pool, base.block_table, 7, ctx - 1, 1, range(L))
    q = torch.empty((L, 1, m, d), dtype=torch.bfloat16, device="cuda")
    k = torch.empty((L, 1, g, d), dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    sd.fill_queries(q, 7, range(L), [ctx])
    sd.fill_new_kv(k, v, 7, range(L), [ctx - 1])
    out = torch.empty((L, 1, m, d), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    _, ws_bytes = d200.query_sizes(cfg)
    for deep in (0, 1):
        print("max active clusters (deep=%d):" % deep,
              {cs: lib.delta_debug_cluster_occupancy(deep, cs) for cs in (2, 4, 8, 12, 16)})
    tunes = os.environ.get("PROBE_TUNES", "auto").split(";")
    for tune in tunes:
        if tune == "auto":
            os.environ.pop("DELTA_TUNE", None)
        else:
            os.environ["DELTA_TUNE"] = tune
        st = d200.DeltaStack(cfg, base.kv_pool, base.block_table,
                             torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda"))
        st.set_seq_lens([ctx - 1])
        with torch.cuda.stream(s):
            st.decode_step(q, k, v, out, stream=s)
        s.synchronize()
        read()
        print(f"########## tune: {tune}")
        for name, fn in (("FULL layer 0", lambda: st.decode_layer(0, q[0], out[0], stream=s)),
                         ("SPARSE layer 3", lambda: st.decode_layer(3, q[3], out[3], stream=s))):
            for rep in range(2):
                with torch.cuda.stream(s):
                    fn()
                s.synchronize()
                tr_ = read()
                report(f"{name} rep {rep}", tr_)
                smid_report(0 if name.startswith("FULL") else 3, 128 if name.startswith("FULL") else 88, tr_)
                if os.environ.get("PROBE_CLUSTERS"):
                    per_cluster(tr_[0] if name.startswith("FULL") else tr_[3])
            if os.environ.get("PROBE_TILES"):
                print(f"   tiles of {name}:")
                tiles()
        # back-to-back: the step's own sequence, eager (timed with events too)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(s):
            ev[0].record(s)
            for l in range(3, 16):
                st.decode_layer(l, q[l], out[l], stream=s)
            ev[1].record(s)
        s.synchronize()
        report(f"SPARSE layer 15 after 3..14 back to back ({ev[0].elapsed_time(ev[1]) * 1e3 / 13:.2f} us/layer)",
               read())
        assert st.get_error() == 0
        st.set_seq_lens([ctx - 1])
        reps = 20
        with torch.cuda.stream(s):
            st.decode_step(q, k, v, out, stream=s)
            s.synchronize()
            for _ in range(3):
                st.set_seq_lens([ctx - 1])
            ev[0].record(s)
            for _ in range(reps):
                st.decode_layer(0, q[0], out[0], stream=s)
            ev[1].record(s)
        s.synchronize()
        print(f"   FULL layer eager back-to-back: {ev[0].elapsed_time(ev[1]) * 1e3 / reps:.2f} us")
        read()
        # graph-captured step (prewait + early trigger): per-layer timeline of the last replay
        st.set_seq_lens([ctx - 1])
        with torch.cuda.stream(s):
            for _ in range(3):
                st.set_seq_lens([ctx - 1])
                st.decode_step(q, k, v, out, stream=s)
        s.synchronize()
        tr = read()
        t0 = tr[:, :, 0][tr[:, :, 0] > 0].min()
        print("   graph step timeline (us from first CTA entry):  layer: entry_min pdl_med data_med loop_med "
              "loop_max push_med sync_med sync_max out_max epi_end")
        for l in list(range(L)) + [32 + d for d in delta]:
            if l >= 32:
                t = tr[l]
                live = t[:, 0] > 0
                if live.any():
                    t = t[live]
                    g = lambda k, fn: (fn(t[:, k][t[:, k] > 0]) - t0) / 1e3 if (t[:, k] > 0).any() else float("nan")
                    print(f"   select L{l - 32}: entry {g(0, np.min):7.2f} waited {g(1, np.max):7.2f} phaseA_done "
                          f"{g(2, np.max):7.2f} elected {g(3, np.max):7.2f} radix_done {g(4, np.max):7.2f} "
                          f"plan_done {g(5, np.max):7.2f} | keys {g(6, np.max):7.2f} passes {g(7, np.max):7.2f} "
                          f"{g(8, np.max):7.2f} {g(9, np.max):7.2f} {g(10, np.max):7.2f} | staged {g(11, np.max):7.2f}")
                continue
            t = tr[l]
            live = t[:, 0] > 0
            if not live.any():
                continue
            t = t[live]
            f = lambda k, fn: (fn(t[:, k][t[:, k] > 0]) - t0) / 1e3 if (t[:, k] > 0).any() else float("nan")
            print(f"   L{l:2d}: {f(0, np.min):7.2f} {f(1, np.median):7.2f} {f(2, np.median):7.2f} "
                  f"{f(3, np.median):7.2f} {f(3, np.max):7.2f} {f(5, np.median):7.2f} {f(7, np.median):7.2f} "
                  f"{f(7, np.max):7.2f} {f(9, np.max):7.2f} {f(6, np.max):7.2f}")


def tiles():
    """Per-tile event times (us) of CTA (0,0,0) of the last traced umma launch."""
    t = np.zeros(64 * 8, np.uint64)
    assert lib.delta_trace_read_tiles(t.ctypes.data_as(ctypes.c_void_p)) == 0
    t = t.reshape(64, 8).astype(np.int64)
    t0 = t[0, 0]
    print("   tile: tma_issued full_seen qk_issued s_seen p_done pv_issued (us from tile-0 TMA issue)")
    for i in range(40):
        r = [(x - t0) / 1e3 if x > 0 else float("nan") for x in t[i, :6]]
        print(f"   {i:3d}: " + " ".join(f"{v:8.2f}" for v in r))


if __name__ == "__main__":
    main()
