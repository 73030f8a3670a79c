import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import paper_1705_01598_b200 as tt, tt_workloads as wl
cs={c.name:c for c in wl.s3_random(per_cell=1)}
for nm in ['S3_r9_x1_e4_0','S3_r4_x5_e4_0','S3_r9_x15_e4_0','S3_r11_x1_e4_0']:
    c=cs[nm]
    for sd in (0,1,-1):
        j=tt.Plan(c.dims,c.perm,c.esize,slot_dims=sd).describe()
        print(nm, sd, j['threads'], j['grid'], j['smem'], j['tile'].get('sd'))
