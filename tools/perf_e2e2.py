"""Stage timing of the overlapped e2e path (bench.run_e2e): ref H2D, index build, reads H2D (side
stream, overlapped with the build), pipelined seeding with streamed D2H; plus raw copy rates."""
import ctypes, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
from paper_2211_08157_b200 import _lib
cfg, pattern, k, w = bench.make_inputs('human', 1.0, 0)
href = torch.from_numpy(cfg.ref).pin_memory(); hroff = torch.from_numpy(cfg.ref_offsets).pin_memory()
hreads = torch.from_numpy(cfg.reads.seq).pin_memory(); hroffs = torch.from_numpy(cfg.reads.offsets).pin_memory()
n = cfg.reads.n
dref = torch.empty_like(href, device='cuda'); droff = torch.empty_like(hroff, device='cuda')
dreads = torch.empty_like(hreads, device='cuda'); droffs = torch.empty_like(hroffs, device='cuda')
L = _lib.load()
prm = _lib.GodParams(pattern.encode(), k, w); cut = _lib.GodCutoff(0, cfg.cutoff[0], cfg.cutoff[1], 0)
main = torch.cuda.current_stream(); side = torch.cuda.Stream()
stream = ctypes.c_void_p(main.cuda_stream)
need = ctypes.c_uint64(0); vp = ctypes.c_void_p
cap = 180_000_000
an_host = torch.empty(cap * 4 + 4, dtype=torch.uint32).pin_memory()
ao_host = torch.empty(n + 1, dtype=torch.uint64).pin_memory(); ph_host = torch.empty(n, dtype=torch.uint8).pin_memory()
big = torch.empty(cap * 4, dtype=torch.uint32, device='cuda')
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dref.copy_(href, non_blocking=True); droff.copy_(hroff, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    ev = torch.cuda.Event(); ev.record(main); side.wait_event(ev)
    with torch.cuda.stream(side):
        dreads.copy_(hreads, non_blocking=True); droffs.copy_(hroffs, non_blocking=True)
    h = ctypes.c_void_p(0)
    _lib.check(L.god_build_index(ctypes.byref(prm), vp(dref.data_ptr()), vp(droff.data_ptr()), 1, ctypes.byref(cut), ctypes.byref(h), stream))
    t2 = time.perf_counter()
    side.synchronize(); t3 = time.perf_counter()
    main.wait_stream(side)
    _lib.check(L.god_seed_reads(h, vp(dreads.data_ptr()), vp(droffs.data_ptr()), n, _lib.PHASE_SELECT, vp(ph_host.data_ptr()), 16,
                                vp(an_host.data_ptr()), vp(ao_host.data_ptr()), cap, ctypes.byref(need), stream))
    torch.cuda.synchronize(); t4 = time.perf_counter()
    L.god_index_free(h)
    # raw D2H of the same anchor bytes
    nb = need.value * 4
    torch.cuda.synchronize(); t5 = time.perf_counter()
    an_host[:nb].copy_(big[:nb], non_blocking=True); torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"it {it}: ref H2D {1e3*(t1-t0):.1f}  build(+reads H2D) {1e3*(t2-t1):.1f}  reads H2D done +{1e3*(t3-t2):.1f}  "
          f"seed+D2H {1e3*(t4-t3):.1f}  total {1e3*(t4-t0):.1f} ms; raw D2H {need.value*16/1e9:.2f} GB in {1e3*(t6-t5):.1f} ms", flush=True)
