// Unity translation unit of libleanot_b200.so (one TU so the exp table symbol
// and the template instantiations exist exactly once; no -rdc needed).
#include "leanot_sweep.cu"
#include "leanot_solver.cu"
#include "leanot_bary.cu"
#include "leanot_sinkhorn.cu"
#include "leanot_dense.cu"
#include "leanot_sep.cu"
#include "leanot_persist.cu"
#include "leanot_fused.cu"
#include "leanot_sr.cu"
