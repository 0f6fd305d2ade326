"""Time the e2e path with pinned host buffers through the C ABI: index build streamed / not streamed,
then the pipelined compact seeding, each by wall clock around the synchronous call."""
import ctypes, os, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench, synth
import paper_2211_08157_b200 as god
from paper_2211_08157_b200 import _lib
scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
cfg, pattern, k, w = bench.make_inputs('human', scale, 0)
href = torch.from_numpy(cfg.ref).pin_memory(); hroff = torch.from_numpy(cfg.ref_offsets).pin_memory()
hreads = torch.from_numpy(cfg.reads.seq).pin_memory(); hroffs = torch.from_numpy(cfg.reads.offsets).pin_memory()
n = cfg.reads.n
L = _lib.load()
prm = _lib.GodParams(pattern.encode(), k, w); cut = _lib.GodCutoff(0, cfg.cutoff[0], cfg.cutoff[1], 0)
stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
need = ctypes.c_uint64(0); vp = ctypes.c_void_p
cap = int(180e6 * scale) + 1024
an_host = torch.empty(cap * 2 + 4, dtype=torch.uint32).pin_memory()
ao_host = torch.empty(n + 1, dtype=torch.uint64).pin_memory(); ph_host = torch.empty(n, dtype=torch.uint8).pin_memory()
dref = torch.empty_like(href, device='cuda')
for chunk in sys.argv[2:] or ["", "0"]:
    if chunk == "":
        os.environ.pop("GOD_STREAM_CHUNK_BYTES", None)
    else:
        os.environ["GOD_STREAM_CHUNK_BYTES"] = chunk
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); h = ctypes.c_void_p(0)
        _lib.check(L.god_build_index(ctypes.byref(prm), vp(href.data_ptr()), vp(hroff.data_ptr()), 1, ctypes.byref(cut), ctypes.byref(h), stream))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        _lib.check(L.god_seed_reads_compact(h, vp(hreads.data_ptr()), vp(hroffs.data_ptr()), n, _lib.PHASE_SELECT, vp(ph_host.data_ptr()), 16,
                                    vp(an_host.data_ptr()), vp(ao_host.data_ptr()), cap, ctypes.byref(need), stream))
        torch.cuda.synchronize(); t2 = time.perf_counter()
        L.god_index_free(h); torch.cuda.synchronize(); t3 = time.perf_counter()
        dref.copy_(href, non_blocking=True); torch.cuda.synchronize(); t4 = time.perf_counter()
        print(f"chunk={chunk!r} it {it}: build {1e3*(t1-t0):.1f} ms  seed {1e3*(t2-t1):.1f} ms  free {1e3*(t3-t2):.1f} ms  plain ref copy {1e3*(t4-t3):.1f} ms  anchors {need.value}", flush=True)
