# sustained samples/s of a BASELINE config over launch shapes: python tools/sweep_cfg.py 1 "128,2;128,4"
import sys; sys.path.insert(0,'.')
import paper_1910_11039_b200 as ebc
c=int(sys.argv[1])
if c==1: g=ebc.gen_erdos_renyi(10000,50000,1)
elif c==2: g=ebc.gen_rmat(20,16,seed=2)
elif c==3: g=ebc.gen_grid(2000,2000,0.05,0.001,3)
elif c==4: g=ebc.gen_rmat(24,16,seed=4)
elif c==14: g=ebc.gen_rmat(14,16,seed=2)
elif c==17: g=ebc.gen_rmat(17,16,seed=2)
elif c==100: g=ebc.gen_erdos_renyi(1000000,8000000,1)
elif c==101: g=ebc.gen_grid(300,300,0.05,0.001,3)
g=g.largest_connected_component()
N={1:400000,2:400000,3:60000,4:100000,14:400000,17:400000,100:200000,101:200000}[c]
for sh in sys.argv[2].split(';'):
    b,i=(int(x) for x in sh.split(','))
    s=ebc.Sampler(g, ebc.RunConfig(block_threads=b, items_per_thread=i)); inf=s.info()
    s.sample(7,0,N//4); s.sync()
    s.mark(0); s.sample(7,N,N); s.mark(1); ms=s.elapsed_ms(0,1)
    print(f"config {c} block {b} items {i} slots {inf['slots']}: {N/ms*1e3:.0f} samples/s", flush=True)
    s.close()
