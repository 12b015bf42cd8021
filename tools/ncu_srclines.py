"""Per-CUDA-source-line warp instruction counts of one kernel of an ncu report
captured with --import-source on (SourceCounters section), plus the SASS opcode mix:
    python tools/ncu_srclines.py report.ncu-rep [kernel index]"""
import csv,sys,subprocess,collections,io
rep=sys.argv[1]; which=int(sys.argv[2]) if len(sys.argv)>2 else 0
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','cuda,sass'],capture_output=True,text=True).stdout
# split into kernels by "Function Name"
blocks=[];cur=None
for line in out.splitlines():
    if line.startswith('"File Path"'):
        continue
    if line.startswith('"Function Name"'):
        cur=[line];blocks.append(cur);continue
    if cur is not None: cur.append(line)
print(len(blocks),'kernel blocks')
b=blocks[which]
print(b[0])
r=list(csv.reader(io.StringIO("\n".join(b[1:]))))
hdr=r[0]
ie=hdr.index('Instructions Executed')
lines=[];sass=collections.Counter();tot=0
curline=None
for x in r[1:]:
    if len(x)<=ie: continue
    if x[0]!='':
        curline=(x[0],x[1]); lines.append([x[0],x[1],(int(x[ie]) if x[ie].isdigit() else 0)])
    else:
        op=x[3].strip().split()
        if op:
            o=op[1] if op[0].startswith('@') else op[0]
            sass[o.split('.')[0]]+=(int(x[ie]) if x[ie].isdigit() else 0)
tot=sum(l[2] for l in lines)
print('total warp inst',tot)
# opcode shares relative to the per-line total (a SASS row listed under several
# inlined source lines counts once per line)
print(', '.join(f"{o}:{n*100/tot:.1f}" for o,n in sass.most_common(24)))
lines.sort(key=lambda l:-l[2])
for l in lines[:45]: print(f"{l[2]*100/tot:5.1f}% {l[0]:>5}: {l[1].strip()[:120]}")
