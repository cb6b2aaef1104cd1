import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
fname=None;hdr=None;out=[]
for r in rows:
    if len(r)==2 and r[0]=="File Path": fname=r[1].split("/")[-1]
    elif r and r[0]=="Line No": hdr=r
    elif hdr and len(r)==len(hdr) and r[0]:
        try: out.append((fname,int(r[0]),float(r[4] or 0),float(r[7] or 0)))
        except: pass
T=sum(o[2] for o in out); E=sum(o[3] for o in out)
ranges=[tuple(map(int,x.split('-'))) for x in sys.argv[2:]]
for a,b in ranges:
    s=sum(o[2] for o in out if o[0]=='pcg_cl.cuh' and a<=o[1]<=b); e=sum(o[3] for o in out if o[0]=='pcg_cl.cuh' and a<=o[1]<=b)
    print(f"{a}-{b}: stall {s/T:.3f} inst {e/E:.3f}")
print("other files: stall %.3f inst %.3f"%(sum(o[2] for o in out if o[0]!='pcg_cl.cuh')/T, sum(o[3] for o in out if o[0]!='pcg_cl.cuh')/E))
