import json,sys
recs=json.load(open(sys.argv[1]))
from collections import defaultdict
byw=defaultdict(list)
for r in recs: byw[r['workload']].append(r)
bytes_={'R':67371008,'G':235175936,'A':67174400,'Q':268566528,'L':33947648}
for w,rs in byw.items():
    ok=[r for r in rs if r['latency_us'] and not r['error'] and r['ff_ok'] is not False]
    ok.sort(key=lambda r:r['latency_us'])
    print(w,len(rs),'ok',len(ok),'ffbad',sum(r['ff_ok'] is False for r in rs),'err',sum(bool(r['error']) for r in rs))
    for r in ok[:int(sys.argv[2]) if len(sys.argv)>2 else 3]:
        print('   %.2f us %.0f GB/s %.0f%%'%(r['latency_us'],bytes_[w]/r['latency_us']/1e3, bytes_[w]/r['latency_us']/1e3/6547.5*100), r.get('timing'), r['params'], r['mapping'], r['plan']['summary'][:150])
