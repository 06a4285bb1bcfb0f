// comm.cu — multi-GPU row-block sharding plumbing (NCCL).
#include "../../include/potgpu.h"

extern "C" {
int potgpu_comm_unique_id(unsigned char*) { return POTGPU_ERR_UNSUPPORTED; }
int potgpu_comm_init(potgpu_ctx*, int, int, const unsigned char*) { return POTGPU_ERR_UNSUPPORTED; }
}
