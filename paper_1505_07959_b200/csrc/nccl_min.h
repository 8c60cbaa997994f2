// Minimal NCCL ABI declarations (types/enums of nccl.h 2.x).  The library resolves the NCCL entry
// points at run time (dlopen of the libnccl.so.2 torch already loaded), so no link-time NCCL
// dependency exists and only one NCCL ever lives in the process.
#pragma once
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0, ncclMax = 2 } ncclRedOp_t;
