"""Discrete-event model of host-path (e2e) schedules on the B200 box: one H2D,
one D2H and one compute queue; PCIe 5 at 55.5/56.8 GB/s one-way and 34 GB/s
in total when both directions run (tools/pcie_probe.py).  Used to choose the
schedule in csrc/capi.cu:host_path."""
# Discrete simulation of host-path schedules: one H2D queue, one D2H queue, one compute queue.
# Bandwidths GB/s; duplex: when both copy directions are active each runs at DUP/2.
H2D, D2H, DUP = 55.5, 56.8, 34.0
M = N = K = 8192
TF = 35.6e12
def simulate(ops):
    # ops: list of (queue, name, amount, deps) ; queue in {'h','d','c'}; amount bytes or flops
    import heapq
    done = {}
    t = 0.0
    pending = {q: [o for o in ops if o[0] == q] for q in 'hdc'}
    cur = {q: None for q in 'hdc'}  # (name, remaining, start)
    while any(pending[q] or cur[q] for q in 'hdc'):
        # start ops whose deps are done
        for q in 'hdc':
            if cur[q] is None and pending[q]:
                op = pending[q][0]
                if all(d in done and done[d] <= t + 1e-12 for d in op[3]):
                    pending[q].pop(0)
                    cur[q] = [op[1], op[2]]
        active = {q for q in 'hdc' if cur[q]}
        if not active:
            # advance to next dep completion (should not happen)
            raise RuntimeError("deadlock")
        rate = {}
        both = 'h' in active and 'd' in active
        rate['h'] = (DUP / 2 if both else H2D) * 1e9
        rate['d'] = (DUP / 2 if both else D2H) * 1e9
        rate['c'] = TF
        dt = min(cur[q][1] / rate[q] for q in active)
        t += dt
        for q in list(active):
            cur[q][1] -= dt * rate[q]
            if cur[q][1] <= 1e-6:
                done[cur[q][0]] = t
                cur[q] = None
    return t

def panel_major(P=8, kchunk_first=0, defer_d2h=False):
    w = N // P
    ops = []
    if kchunk_first:
        ch = K // kchunk_first
        ops.append(('h', 'C0', 8*M*w, []))
        for kc in range(kchunk_first):
            ops.append(('h', f'A{kc}', 8*M*ch, []))
            ops.append(('h', f'B0_{kc}', 8*ch*w, []))
            ops.append(('c', f'c0_{kc}', 2*M*w*ch, [f'A{kc}', f'B0_{kc}', 'C0'] + ([f'c0_{kc-1}'] if kc else [])))
        last0 = f'c0_{kchunk_first-1}'
        adeps = [f'A{kc}' for kc in range(kchunk_first)]
    else:
        ops.append(('h', 'A', 8*M*K, []))
        ops.append(('h', 'C0', 8*M*w, [])); ops.append(('h', 'B0', 8*K*w, []))
        ops.append(('c', 'c0', 2*M*w*K, ['A', 'C0', 'B0']))
        last0 = 'c0'; adeps = ['A']
    comp = [last0]
    for p in range(1, P):
        ops.append(('h', f'C{p}', 8*M*w, [])); ops.append(('h', f'B{p}', 8*K*w, []))
        ops.append(('c', f'c{p}', 2*M*w*K, adeps + [f'C{p}', f'B{p}', comp[-1]]))
        comp.append(f'c{p}')
    hl = [o[1] for o in ops if o[0]=='h'][-1]
    for p in range(P):
        ops.append(('d', f'D{p}', 8*M*w, [comp[p]] + ([hl] if defer_d2h else [])))
    return ops

for P in (8, 16):
    for kf in (0, 8, 16):
        for dd in (False, True):
            t = simulate(panel_major(P, kf, dd))
            print(f"P={P} kchunk_first={kf} defer_d2h={dd}: {t*1e3:.1f} ms  -> {2*M*N*K/t/1e12:.1f} TF")

def kouter_c_at_end(P=8, KC=8, final_kc=1):
    # P(all) = A*B accumulated over k-chunks from zero; C uploaded after A/B;
    # final `final_kc` chunks processed panel by panel followed by +C and D2H.
    w = N // P; ch = K // KC
    ops = []
    for kc in range(KC):
        ops.append(('h', f'A{kc}', 8*M*ch, []))
        ops.append(('h', f'B{kc}', 8*ch*N, []))
    ops.append(('h', 'C', 8*M*N, []))
    prev = []
    for kc in range(KC - final_kc):
        ops.append(('c', f'k{kc}', 2*M*N*ch, [f'A{kc}', f'B{kc}'] + prev)); prev = [f'k{kc}']
    last = prev
    for p in range(P):
        deps = [f'A{kc}' for kc in range(KC)] + [f'B{kc}' for kc in range(KC)] + ['C'] + last
        ops.append(('c', f'f{p}', 2*M*w*ch*final_kc, deps)); last = [f'f{p}']
        ops.append(('d', f'D{p}', 8*M*w, [f'f{p}', 'C']))
    return ops

def kouter_c_first_sweep(P=8, KC=8):
    # acc-from-C: chunk 0 per panel needs C_p; chunks >= 1 k-outer; final chunk panel-major + D2H
    w = N // P; ch = K // KC
    ops = [('h', 'A0', 8*M*ch, []), ('h', 'B0', 8*ch*N, [])]
    prev = []
    for p in range(P):
        ops.append(('h', f'C{p}', 8*M*w, []))
        ops.append(('c', f'c0_{p}', 2*M*w*ch, ['A0', 'B0', f'C{p}'] + prev)); prev = [f'c0_{p}']
    for kc in range(1, KC):
        ops.append(('h', f'A{kc}', 8*M*ch, [])); ops.append(('h', f'B{kc}', 8*ch*N, []))
    for kc in range(1, KC - 1):
        ops.append(('c', f'k{kc}', 2*M*N*ch, [f'A{kc}', f'B{kc}'] + prev)); prev = [f'k{kc}']
    for p in range(P):
        ops.append(('c', f'f{p}', 2*M*w*ch, [f'A{KC-1}', f'B{KC-1}'] + prev)); prev = [f'f{p}']
        ops.append(('d', f'D{p}', 8*M*w, [f'f{p}', f'B{KC-1}']))
    return ops

for P in (8, 16, 32):
    for KC in (8, 16):
        for fk in (1, 2, 4):
            if fk >= KC: continue
            t = simulate(kouter_c_at_end(P, KC, fk))
            print(f"C-at-end P={P} KC={KC} final={fk}: {t*1e3:.1f} ms -> {2*M*N*K/t/1e12:.1f} TF")
    for KC in (8, 16):
        t = simulate(kouter_c_first_sweep(P, KC))
        print(f"C-first-sweep P={P} KC={KC}: {t*1e3:.1f} ms -> {2*M*N*K/t/1e12:.1f} TF")

def group_first(g0_frac, P_rest=4, KC=8):
    w0 = int(N * g0_frac) // 128 * 128; rest = N - w0
    wr = rest // P_rest if P_rest else 0
    ch = K // KC
    ops = [('h', 'C0', 8*M*w0, [])]
    prev = []
    for kc in range(KC):
        ops.append(('h', f'A{kc}', 8*M*ch, [])); ops.append(('h', f'B0_{kc}', 8*ch*w0, []))
        ops.append(('c', f'c0_{kc}', 2*M*w0*ch, [f'A{kc}', f'B0_{kc}', 'C0'] + prev)); prev = [f'c0_{kc}']
    comp = [prev[0]]
    adeps = [f'A{kc}' for kc in range(KC)]
    for p in range(1, P_rest + 1):
        ops.append(('h', f'B{p}', 8*K*wr, [])); ops.append(('h', f'C{p}', 8*M*wr, []))
        ops.append(('c', f'c{p}', 2*M*wr*K, adeps + [f'B{p}', f'C{p}', comp[-1]])); comp.append(f'c{p}')
    hl = [o[1] for o in ops if o[0]=='h'][-1]
    ops.append(('d', 'D0', 8*M*w0, [comp[0], hl]))
    for p in range(1, P_rest + 1):
        ops.append(('d', f'D{p}', 8*M*wr, [comp[p], hl]))
    return ops
for f in (0.125, 0.25, 0.375, 0.5, 0.625):
    for pr in (2, 4, 8):
        for KC in (8, 16):
            t = simulate(group_first(f, pr, KC))
            print(f"group0={f} rest_panels={pr} KC={KC}: {t*1e3:.1f} ms -> {2*M*N*K/t/1e12:.1f} TF")
