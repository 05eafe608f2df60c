"""Shared-memory bank model of bp_apply_kernel (apply.cu) used to choose the
per-column pads col_pad(kind, p, KC): every phase access of a CTA's KC
element columns, 8-byte words on 16 banks, each half-warp a separate request
(wf_half: the largest number of distinct words on one bank; the whole-warp
variant wf mispredicted BP5 p = 2). Dev tool.
    python tools/bank_model.py        # pads per default (kind, p, KC)
"""
import itertools
def best_stride(N,Q,base,kind):
    def cost(S):
        tot=0; nact=N*Q
        for h0 in range(0,nact,16):
            words=set()
            for t in range(h0,min(h0+16,nact)):
                i=t%N; c=t//N
                words.add(c*S+i if kind==0 else i*S+c*Q)
            cnt={}
            for w in words: cnt[w%16]=cnt.get(w%16,0)+1
            tot+=max(cnt.values())
        return tot
    return min(range(base,base+16), key=lambda S:(cost(S),S))
def wf(addrs):  # addrs: list of word addresses (None = inactive)
    ws=set(a for a in addrs if a is not None)
    if not ws: return 0
    cnt={}
    for w in ws: cnt[w%16]=cnt.get(w%16,0)+1
    return max(max(cnt.values()), (len(ws)+15)//16)
def model(P,KIND,KC,CBpad=0,GSpad=0,verbose=False):
    N=P+1; Q=P+1 if KIND==2 else P+2; QQ=Q*Q
    FA=1 if KIND==0 else 2; FB=1 if KIND==0 else 3
    SA_CS=best_stride(N,Q,N*N,0); SB_IS=best_stride(N,Q,Q*Q,1)
    SA_SIZE=FA*Q*SA_CS; SB_SIZE=FB*N*SB_IS
    CB=(SA_SIZE+SB_SIZE+1)//2*2 + CBpad
    COMP=1 if KIND==0 else 6
    GS=(COMP*Q**3+1)//2*2 + GSpad
    ZI=KC*N*N; YI=KC*N*Q; XI=KC*QQ; NT=((XI+31)//32)*32
    total=0; parts={}
    def acc(name, fn, nitems, reps):
        nonlocal total
        s=0
        for w0 in range(0,NT,32):
            if w0>=nitems: continue
            for r in reps:
                addrs=[fn(t,*r) if t<nitems else None for t in range(w0,w0+32)]
                s+=wf(addrs)
        parts[name]=s; total+=s
    # phase Z writes SA[kz*CB + (f*Q+c)*SA_CS + pz]
    acc('Zw', lambda t,f,c: (t//(N*N))*CB + (f*Q+c)*SA_CS + t%(N*N), ZI, [(f,c) for f in range(FA) for c in range(Q)])
    # phase Y reads SA[ky*CB + (f*Q+c)*SA_CS + j*N + i]
    def yr(t,f,j):
        ky=t//(N*Q); rem=t%(N*Q); i=rem%N; c=rem//N
        return ky*CB+(f*Q+c)*SA_CS+j*N+i
    acc('Yr', yr, YI, [(f,j) for f in range(FA) for j in range(N)])
    def yw(t,f,b):
        ky=t//(N*Q); rem=t%(N*Q); i=rem%N; c=rem//N
        return ky*CB+SA_SIZE+f*N*SB_IS+i*SB_IS+c*Q+b
    acc('Yw', yw, YI, [(f,b) for f in range(FB) for b in range(Q)])
    def xr(t,f,i):
        kx=t//QQ; pp=t%QQ
        return kx*CB+SA_SIZE+(f*N+i)*SB_IS+pp
    acc('Xr', xr, XI, [(f,i) for f in range(FB) for i in range(N)])
    acc('Xw', xr, XI, [(f,i) for f in range(FB) for i in range(N)])
    def xg(t,m,a):
        kx=t//QQ; pp=t%QQ
        return 100000+kx*GS+m*Q*QQ+a*QQ+pp
    acc('XG', xg, XI, [(m,a) for m in range(COMP) for a in range(Q)])
    acc("Y'r", yw, YI, [(f,b) for f in range(FB) for b in range(Q)])
    acc("Y'w", yr, YI, [(f,j) for f in range(FA) for j in range(N)])
    acc("Z'r", lambda t,f,c: (t//(N*N))*CB + (f*Q+c)*SA_CS + t%(N*N), ZI, [(f,c) for f in range(FA) for c in range(Q)])
    return total, parts, CB, GS
def wf_half(addrs):
    tot=0
    for h in (0,16):
        ws=set(a for a in addrs[h:h+16] if a is not None)
        if not ws: continue
        cnt={}
        for w in ws: cnt[w%16]=cnt.get(w%16,0)+1
        tot+=max(cnt.values())
    return tot

def table(all_kc=False):
    """col_pad codes (cb_pad * 100 + gs_pad): the default work splits (sk_default),
    or (--table) every p <= 6 and KC = 2..8 (apply.cu kColPad; several minutes)."""
    global wf
    cfgs={0:{3:4,4:5,5:3,8:2},1:{1:7,2:2,3:3,4:2},2:{1:8,2:3,3:2,4:3,5:2,6:2}}
    if all_kc:
        cfgs={k:{(P,KC):None for P in range(1,7) for KC in range(2,9) if KC*(P+1 if k==2 else P+2)**2<=1024} for k in range(3)}
    full=wf
    for kind,d in cfgs.items():
        for key in d:
            P,KC=key if all_kc else (key,d[key])
            res=[]
            for c in range(16):
                for g in range(0,16,2):
                    wf=wf_half; h=model(P,kind,KC,c,g)[0]
                    wf=full; f=model(P,kind,KC,c,g)[0]
                    res.append((h,f,c,g))
            base=[r for r in res if r[2]==0 and r[3]==0][0]
            best=min(res)
            print(kind,P,KC,'half-warp wavefronts',base[0],'->',best[0],'code',best[2]*100+best[3] if best[0]<base[0] else 0)


def u_staging(P, KC, UP):
    """u staging slabs (cp.async write, phase-Z read, epilogue read): pencil pz
    of column kz at kz (2 n^3 + UP) + k n^2 + pz (apply.cu u_pad)."""
    N = P + 1; ZI = KC * N * N; s = 0
    for w0 in range(0, ((ZI + 31) // 32) * 32, 32):
        for k in range(N):
            s += wf([(t // (N * N)) * (2 * N ** 3 + UP) + k * N * N + t % (N * N) if t < ZI else None
                     for t in range(w0, w0 + 32)])
    return 3 * s


if __name__=='__main__':
    import sys
    table('--table' in sys.argv)
