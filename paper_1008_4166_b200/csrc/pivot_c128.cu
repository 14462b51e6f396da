// Second translation unit of the round-1 cluster pivot kernel: the
// complex128 instantiations (see the note at the top of pivot.cu).
#define HJB_PIVOT_CPLX_TU 1
#include "pivot.cu"
