"""Instruction count and top SASS lines of an ncu report by warp-stall samples.
usage: python sass_hot.py report.ncu-rep [min percent]"""
import csv,sys,subprocess,io,re
rep=sys.argv[1]; thr=float(sys.argv[2]) if len(sys.argv)>2 else 0.5
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source=sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(io.StringIO(out)))
h=rows[1]
tot=0; data=[]; itot=0
for i,r in enumerate(rows[2:]):
    d=dict(zip(h,r))
    try: v=float(d['Warp Stall Sampling (All Samples)']); ie=float(d['Instructions Executed'])
    except: continue
    tot+=v; itot+=ie; data.append((v,i,ie,d['Source'].strip()))
print('samples',tot,'warp-instr',itot)
for v,i,ie,s in data:
    if v>tot*thr/100: print(f'{100*v/tot:5.1f}% {i:5d} {ie:10.0f} {s}')
