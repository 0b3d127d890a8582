/* fk_cuda.h — entry points only the CUDA backend (libfk_cuda.so) exports. */
#ifndef FK_CUDA_H_
#define FK_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Writes "<name> sm_<cc> SMs=<n> L2=<bytes>" for the current device; returns the status. */
int32_t fk_cuda_device_info(char* buf, size_t cap);
/* Fused-kernel launches enqueued by this process so far (all executors). */
uint64_t fk_cuda_kernel_launch_count(void);
/* Name of the kernel the last fused execute on this thread launched
   ("fk_direct", "fk_resample_sep", "fk_resample", "fk_transform_generic"), or "". */
const char* fk_cuda_last_kernel(void);

#ifdef __cplusplus
}
#endif

#endif /* FK_CUDA_H_ */
