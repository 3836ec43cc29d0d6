import random, sys
import os; sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from fnv_bitslice_gen import gen_network
P=(1<<40)+0x1b3; M64=(1<<64)-1; M32=(1<<32)-1
def fnv(bs,h=0xcbf29ce484222325):
    for b in bs: h=((h^b)*P)&M64
    return h
def t8x8(x):
    t=(x^(x>>7))&0x00AA00AA00AA00AA; x=x^t^((t<<7)&M64)
    t=(x^(x>>14))&0x0000CCCC0000CCCC; x=x^t^((t<<14)&M64)
    t=(x^(x>>28))&0x00000000F0F0F0F0; x=x^t^((t<<28)&M64)
    return x
def slice32(w):  # w[8] words of 4 bytes -> 8 planes
    xs=[t8x8(w[2*q]|(w[2*q+1]<<32)) for q in range(4)]
    return [sum((((xs[q]>>(8*j))&0xff)<<(8*q)) for q in range(4)) for j in range(8)]
def unslice32(pl):
    w=[0]*8
    for q in range(4):
        x=sum((((pl[j]>>(8*q))&0xff)<<(8*j)) for j in range(8))
        x=t8x8(x); w[2*q]=x&M32; w[2*q+1]=x>>32
    return w
# check transpose convention
for _ in range(100):
    bs=[random.randrange(256) for _ in range(32)]
    w=[sum(bs[4*k+i]<<(8*i) for i in range(4)) for k in range(8)]
    pl=slice32(w)
    for j in range(8):
        for s in range(32): assert (pl[j]>>s)&1==(bs[s]>>j)&1
    assert unslice32(pl)==w
net=gen_network()
def prefx(p):
    p^=(p<<1)&M32; p^=(p<<2)&M32; p^=(p<<4)&M32; p^=(p<<8)&M32; p^=(p<<16)&M32
    return p
PW=[pow(P,32*(31-L),1<<64) for L in range(32)]
PT=[pow(P,k,1<<64) for k in range(33)]
def block(h_in, lanes_bytes, lanes_vm):
    """lanes_bytes[L]: 32 bytes (invalid = 0); lanes_vm[L]: 32-bit valid masks (invalid steps only at the front of the block)."""
    l0=h_in&0xff
    Bp=[slice32([sum(b[4*k+i]<<(8*i) for i in range(4)) for k in range(8)]) for b in lanes_bytes]
    X=[[0]*8 for _ in range(32)]; Lp=[[0]*8 for _ in range(32)]; K=[[0]*8 for _ in range(32)]; envs=[{} for _ in range(32)]
    for j in range(8):
        par=[0]*32; pre=[0]*32
        for L in range(32):
            env=envs[L]; env.update({f"X{i}":X[L][i] for i in range(j)}); env.update({f"K{i}":K[L][i] for i in range(j)})
            for line in net[j]:
                name,expr=line.replace("const uint32_t ","").rstrip(";").split(" = ",1)
                env[name]=eval(expr.replace("0u","0"),{},env)&M32
            G=env[f"G{j}"]
            T=(Bp[L][j]^G)&lanes_vm[L]
            p=prefx(T); pre[L]=(p<<1)&M32; par[L]=p>>31
            X[L][j]=G  # stash G temporarily
        for L in range(32):
            carry=((l0>>j)&1)^(sum(par[:L])&1)
            Lj=pre[L]^(M32 if carry else 0)
            G=X[L][j]
            Lp[L][j]=Lj; X[L][j]=Lj^Bp[L][j]; K[L][j]=X[L][j]&G
    h=0
    first_lane=next((L for L in range(32) if lanes_vm[L]),None)
    if first_lane is None: return h_in
    for L in range(32):
        lw=unslice32(Lp[L]); acc=0
        for s in range(32):
            if not (lanes_vm[L]>>s)&1: continue
            b=lanes_bytes[L][s]; l=(lw[s//4]>>(8*(s%4)))&0xff
            d=b-2*(b&l)
            acc=(acc+d*PT[32-s])&M64
        if L==first_lane:
            sf=(lanes_vm[L]&-lanes_vm[L]).bit_length()-1
            acc=(acc+h_in*PT[32-sf])&M64
        h=(h+acc*PW[L])&M64
    return h
def fnv_blocks(bs,h0=0xcbf29ce484222325):
    N=len(bs)
    if N==0: return h0
    nb=(N+1023)//1024; pad=nb*1024-N
    h=h0
    for B in range(nb):
        lb=[];lv=[]
        for L in range(32):
            b=[];vm=0
            for s in range(32):
                t=B*1024+32*L+s
                if t>=pad: b.append(bs[t-pad]); vm|=1<<s
                else: b.append(0)
            lb.append(b);lv.append(vm)
        h=block(h,lb,lv)
    return h
for n in [0,1,2,31,32,33,100,1023,1024,1025,2500,3933]:
    bs=[random.randrange(256) for _ in range(n)]
    assert fnv(bs)==fnv_blocks(bs),n
print("block model ok")
