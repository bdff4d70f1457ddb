import sys,re,collections
tot=0;n=0;b=collections.defaultdict(lambda:[0,0.0,0])
for l in open(sys.argv[1]):
    m=re.match(r"\[jacobi\] p=(\d+) k=(\d+) sweeps=(\d+) ms=([\d.]+)",l)
    if not m: continue
    p,k,sw,ms=int(m[1]),int(m[2]),int(m[3]),float(m[4]); tot+=ms;n+=1
    key=(k//25)*25; b[key][0]+=1;b[key][1]+=ms;b[key][2]+=sw
print("jacobi calls",n,"total ms",tot)
for k in sorted(b): print(f"k {k:4d}-{k+24}: n={b[k][0]:5d} ms={b[k][1]:9.1f} avg sweeps={b[k][2]/b[k][0]:.1f} avg ms={b[k][1]/b[k][0]:.2f}")
