// Minimal NCCL ABI declarations (types/enums of nccl.h 2.x).  The library resolves the NCCL entry
// points at run time (dlopen of the libnccl.so.2 torch already loaded), so no link-time NCCL
// dependency exists and only one NCCL ever lives in the process.
#pragma once
typedef struct ncclComm* ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0, ncclMax = 2 } ncclRedOp_t;

// ncclConfig_t of nccl.h 2.28 (ncclConfig_v22800; NCCL_CONFIG_INITIALIZER sets size / magic /
// version and leaves every attribute undefined).  Used only when ncclGetVersion() >= 22800.
#include <climits>
#include <cstddef>
typedef struct {
  size_t size;
  unsigned int magic;
  unsigned int version;
  int blocking;
  int cgaClusterSize;
  int minCTAs;
  int maxCTAs;
  const char* netName;
  int splitShare;
  int trafficClass;
  const char* commName;
  int collnetEnable;
  int CTAPolicy;
  int shrinkShare;
  int nvlsCTAs;
  int nChannelsPerNetPeer;
  int nvlinkCentricSched;
} ncclConfig_t;
static inline ncclConfig_t nccl_config_init(int version_code) {
  ncclConfig_t c;
  c.size = sizeof(ncclConfig_t);
  c.magic = 0xcafebeef;
  c.version = (unsigned)version_code;
  c.blocking = c.cgaClusterSize = c.minCTAs = c.maxCTAs = INT_MIN;
  c.netName = nullptr;
  c.splitShare = c.trafficClass = INT_MIN;
  c.commName = nullptr;
  c.collnetEnable = c.CTAPolicy = c.shrinkShare = c.nvlsCTAs = c.nChannelsPerNetPeer = c.nvlinkCentricSched = INT_MIN;
  return c;
}
