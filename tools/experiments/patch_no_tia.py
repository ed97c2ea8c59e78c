import re
p='paper_1907_08467_b200/csrc/cpu.cuh'
s=open(p).read()
s=s.replace("      c.lg[log_len * c.s] = log_entry(3u * now, r, v);\n      ++log_len;","#ifndef CULE_EXP_NO_TIA\n      c.lg[log_len * c.s] = log_entry(3u * now, r, v);\n      ++log_len;\n#endif",1)
s=s.replace("      if (r < 8u) return tia_coll_read(c, r, kPhaseA ? t_phaseA : 3u * now);","#ifndef CULE_EXP_NO_TIA\n      if (r < 8u) return tia_coll_read(c, r, kPhaseA ? t_phaseA : 3u * now);\n#else\n      if (r < 8u) return 0u;\n#endif",1)
open(p,'w').write(s)
p='paper_1907_08467_b200/csrc/kernels.cuh'
s=open(p).read()
s=s.replace("      if (m.log_len || fin) flush_call(","#ifndef CULE_EXP_NO_TIA\n      if (m.log_len || fin) flush_call(",1)
s=s.replace("3u * m.fc, c.ystart, c.gray);\n      m.log_len = 0;","3u * m.fc, c.ystart, c.gray);\n#endif\n      m.log_len = 0;",1)
open(p,'w').write(s)
