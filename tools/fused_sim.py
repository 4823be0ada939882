# CPU model of the fused kernel's ticket / dependency protocol (fused.cuh): checks
# deadlock freedom, exactly-once processing and dependency order under random
# interleavings of CTAs.  usage: python tools/fused_sim.py
import random
def sim(nsig, U, lag, nctas, seed):
    rnd = random.Random(seed)
    SU = sum(U); nticket = (nsig + 2*lag)*SU
    ticket = [0]; done = [[0]*nsig for _ in range(3)]
    processed = {}
    def take():
        while True:
            q = ticket[0]; ticket[0] += 1
            if q >= nticket: return None
            k, r = divmod(q, SU)
            if r < U[2]: p, s = 2, k-2*lag
            elif r - U[2] < U[1]: p, s, r = 1, k-lag, r-U[2]
            else: p, s, r = 0, k, r-U[2]-U[1]
            if 0 <= s < nsig: return [p, s, s*U[p]+r, False]
    def ready(j): return j[0] == 0 or done[j[0]-1][j[1]] >= U[j[0]-1]
    def signal(j): done[j[0]][j[1]] += 1
    # CTA state machine
    ctas = []
    for c in range(nctas):
        ctas.append({'jobs':[None,None], 'pa':None, 'pb':None, 'it':0, 'state':'pro', 'fin':False})
    while True:
        live = [c for c in ctas if not c['fin']]
        if not live: break
        progress = False
        rnd.shuffle(live)
        for c in live:
            st = c['state']
            if st == 'pro':
                if 'j0' not in c: c['j0'] = take()
                j0 = c['j0']
                if j0 is not None:
                    if not ready(j0): continue   # blocking (holds nothing)
                    j0[3] = True
                c['jobs'][0] = j0; c['state'] = 'top'; progress = True; break
            if st == 'top':
                b = c['it'] & 1; J = c['jobs'][b]
                if J is None:
                    for k in ('pa','pb'):
                        if c[k]: signal(c[k]); c[k] = None
                    c['fin'] = True; progress = True; break
                if not J[3]:
                    for k in ('pa','pb'):
                        if c[k]: signal(c[k]); c[k] = None
                    if not ready(J): progress = progress; continue
                    J[3] = True
                c['state'] = 'svc'; progress = True; break
            if st == 'svc':
                b = c['it'] & 1; J = c['jobs'][b]
                if c['pa']: signal(c['pa'])
                c['pa'] = c['pb']; c['pb'] = None
                n = take()
                if n is not None and ready(n): n[3] = True
                c['jobs'][b^1] = n
                key = (J[0], J[2]); assert key not in processed, key
                assert ready(J), ('dependency violated', J)
                processed[key] = 1
                c['pb'] = J; c['it'] += 1; c['state'] = 'top'; progress = True; break
        if not progress:
            return 'DEADLOCK', ticket[0], done
    tot = nsig*sum(U)
    assert len(processed) == tot, (len(processed), tot)
    return 'ok'
CASES = [(2, [274, 243, 274], 1, 148), (64, [274, 243, 274], 1, 148), (64, [274, 243, 274], 1, 3),
         (8, [25, 25, 25], 1, 296), (100, [25, 25, 25], 4, 296), (1, [16, 256, 16], 1, 148),
         (5, [3, 2, 3], 1, 40), (3, [1, 1, 1], 1, 7), (6, [0, 5, 0], 1, 9)]

if __name__ == "__main__":
    for args in CASES:
        for seed in range(20):
            r = sim(*args, seed)
            if r != 'ok':
                print(args, seed, r[0])
                break
        else:
            print(args, 'ok')
