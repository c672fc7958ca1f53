import csv,sys
from collections import OrderedDict
def load(fn):
    rows=[r for r in csv.reader(open(fn)) if len(r)>10]
    hdr=rows[0]; rows=rows[1:]
    I={h:i for i,h in enumerate(hdr)}
    L=OrderedDict()
    for r in rows:
        k=r[I['ID']]
        d=L.setdefault(k,{'name':r[I['Kernel Name']]})
        v=float(r[I['Metric Value']].replace(',',''))
        u=r[I['Metric Unit']]
        m=r[I['Metric Name']]
        if m=='gpu__time_duration.sum':
            v={'ns':1e-3,'nsecond':1e-3,'us':1,'usecond':1,'ms':1e3,'msecond':1e3}.get(u,1)*v
        elif 'bytes' in m:
            v=v*{'byte':1e-9,'Kbyte':1e-6,'Mbyte':1e-3,'Gbyte':1}.get(u,1)
        d[m]=v
    ks=list(L.values())
    idx=[i for i,d in enumerate(ks) if 'k_prep_weights' in d['name']]
    return ks[idx[-1]:] if idx else ks
if __name__=='__main__':
    step=load(sys.argv[1])
    tot=0
    for d in step:
        t=d['gpu__time_duration.sum']; tot+=t
        print(f"{t:8.1f} us tp={d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed',0):5.1f} R={d.get('dram__bytes_read.sum',0):6.3f} W={d.get('dram__bytes_write.sum',0):6.3f} {d['name'][:80]}")
    print('total us', tot)
