// switch_tc_fused.cu -- the v1 tensor-core switch kernel compiled with the fused
// switch + decode epilogue as lsw::v1f; see switch_tc.cu.
#define LSW_TC_FUSED 1
#include "switch_tc.cu"
