// generated: explicit instantiation of the N_mv = 2^13 engine
#include "../tsf_dispatch_impl.cuh"

template struct tsf::Dispatch<13>;
