"""Where the e2e step's extra time goes (GPU box only): the bench's batch
sweep 1..32 at 8192x22016 e3m2, graph-replayed, in variants
  kern      six linears per step, back to back (bench `value`)
  events    + the e2e event structure (fork/join, per-step waits), no copies
  h2d       + the per-step H2D only
  d2h       + the per-step D2H only
  full      H2D + D2H (bench `e2e`)
  early     full, with the wait for step k's upload placed before step
            k-1's last linear (so step boundaries stay kernel -> kernel)
env: STEPS (20), REPS (5)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

ctx = bench.Ctx(0, 1, 0)
torch, L, fpx = ctx.torch, ctx.L, ctx.fpx
dev = ctx.dev
M, K = bench.M_ROWS, bench.K_COLS
steps, reps = int(os.environ.get("STEPS", 20)), int(os.environ.get("REPS", 5))
batches = [1, 2, 4, 8, 16, 32]
p0 = bench.make_packed(ctx, M, K, seed=1)
copies = [p0] + [bench.clone_packed(ctx, p0) for _ in range(2)]
ptrs = [(C.c_void_p * 2)(*[s.data_ptr() for s in cp.streams]) for cp in copies]
splits = {n: fpx.default_split(M, K, n) for n in batches}
ws = torch.zeros(int(max(L.fpx_linear_workspace_size(M, K, K, n, splits[n]) for n in batches)), dtype=torch.uint8,
                 device=dev)
tot_a, tot_c = sum(batches) * K, sum(batches) * M
h_act = bench.page_locked(torch, torch.randn(tot_a).half())
h_out = bench.page_locked(torch, torch.empty(tot_c))
d_act = [torch.randn(tot_a, device=dev).half() for _ in range(2)]
d_out = [torch.empty(tot_c, device=dev) for _ in range(2)]
aoff, coff, a, c = {}, {}, 0, 0
for n in batches:
    aoff[n], coff[n] = a, c
    a += n * K
    c += n * M
s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)


def launch(i, n, par):
    cp = copies[i % 3]
    st = L.fpx_linear(ptrs[i % 3], 2, cp.scales.data_ptr(), M, K, 3, 2, d_act[par][aoff[n]:].data_ptr(), K, n,
                      d_out[par][coff[n]:].data_ptr(), M, splits[n], ws.data_ptr(), ws.numel(), ctx.stream())
    assert st == 0


def launch_zc(i, n):
    """fpx_linear writing C straight into the pinned host buffer (UVA)."""
    cp = copies[i % 3]
    st = L.fpx_linear(ptrs[i % 3], 2, cp.scales.data_ptr(), M, K, 3, 2, d_act[i & 1][aoff[n]:].data_ptr(), K, n,
                      h_out[coff[n]:].data_ptr(), M, splits[n], ws.data_ptr(), ws.numel(), ctx.stream())
    assert st == 0


def variant_zc(h2d):
    def fn():
        main = torch.cuda.current_stream(dev)
        fork = torch.cuda.Event()
        fork.record(main)
        s_h2d.wait_event(fork)
        ran, up = {}, {}
        i = 0
        for k in range(steps):
            par = k & 1
            if k >= 2:
                s_h2d.wait_event(ran[k - 2])
            with torch.cuda.stream(s_h2d):
                if h2d:
                    d_act[par].copy_(h_act, non_blocking=True)
                up[k] = torch.cuda.Event()
                up[k].record(s_h2d)
            main.wait_event(up[k])
            for n in batches:
                launch_zc(i, n)
                i += 1
            ran[k] = torch.cuda.Event()
            ran[k].record(main)
        j1 = torch.cuda.Event()
        j1.record(s_h2d)
        main.wait_event(j1)
    return fn


def variant(h2d, d2h, events, early=False):
    def fn():
        main = torch.cuda.current_stream(dev)
        fork = torch.cuda.Event()
        fork.record(main)
        s_h2d.wait_event(fork)
        s_d2h.wait_event(fork)
        ran, down, up = {}, {}, {}
        i = 0

        def upload(k):
            par = k & 1
            if k >= 2:
                s_h2d.wait_event(ran[k - 2])
            with torch.cuda.stream(s_h2d):
                if h2d:
                    d_act[par].copy_(h_act, non_blocking=True)
                up[k] = torch.cuda.Event()
                up[k].record(s_h2d)

        if early:
            upload(0)
        for k in range(steps):
            par = k & 1
            if events and k >= 2:
                main.wait_event(down[k - 2])
            if events and not early:
                upload(k)
                main.wait_event(up[k])
            elif events and early and k == 0:
                main.wait_event(up[0])
            for j, n in enumerate(batches):
                if events and early and j == len(batches) - 1 and k + 1 < steps:
                    ran_pre = torch.cuda.Event()
                    ran_pre.record(main)
                    ran[k - 1 + 0] = ran.get(k - 1, ran_pre)
                    upload(k + 1)
                    main.wait_event(up[k + 1])
                launch(i, n, par)
                i += 1
            if events:
                ran[k] = torch.cuda.Event()
                ran[k].record(main)
                s_d2h.wait_event(ran[k])
                with torch.cuda.stream(s_d2h):
                    if d2h:
                        h_out.copy_(d_out[par], non_blocking=True)
                    down[k] = torch.cuda.Event()
                    down[k].record(s_d2h)
        if events:
            j1, j2 = torch.cuda.Event(), torch.cuda.Event()
            j1.record(s_h2d)
            j2.record(s_d2h)
            main.wait_event(j1)
            main.wait_event(j2)
    return fn


for name, fnv in [("kern", variant(False, False, False)), ("full", variant(True, True, True)),
                  ("zc_out", variant_zc(False)), ("zc+h2d", variant_zc(True)), ("kern", variant(False, False, False)),
                  ("full", variant(True, True, True)), ("zc+h2d", variant_zc(True))]:
    gr = ctx.capture(fnv)
    for _ in range(2):
        gr.replay()
    ms = ctx.timed(gr, reps) / reps
    print(f"{name:7s} {ms * 1e3 / steps:7.1f} us/step", flush=True)
    del gr
# check: the zero-copy output equals the device output
torch.cuda.synchronize()
ref = d_out[0].cpu()
launch(0, 16, 0)
launch_zc(0, 16)
torch.cuda.synchronize()
print("zc C == device C:", bool(torch.equal(h_out[coff[16]:coff[16] + 16 * M], d_out[0][coff[16]:coff[16] + 16 * M].cpu())))
sys.exit(0)
for name, args in [("kern", (False, False, False)), ("events", (False, False, True)), ("h2d", (True, False, True)),
                   ("d2h", (False, True, True)), ("full", (True, True, True)), ("early", (True, True, True, True)),
                   ("kern", (False, False, False)), ("full", (True, True, True))]:
    gr = ctx.capture(variant(*args))
    for _ in range(2):
        gr.replay()
    ms = ctx.timed(gr, reps) / reps
    print(f"{name:7s} {ms * 1e3 / steps:7.1f} us/step", flush=True)
    del gr
