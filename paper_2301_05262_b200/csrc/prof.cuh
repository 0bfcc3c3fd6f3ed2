#pragma once

#include <cuda_runtime.h>
#include <cstring>

#include "../../include/nsm.h"

namespace nsm {

// RAII scope around one kernel launch (see prof.cu).
class ProfScope {
   public:
    ProfScope(const char* name, cudaStream_t s);
    ~ProfScope();

   private:
    const char* name_;
    cudaStream_t s_;
    cudaEvent_t a_{}, b_{};
    bool on_ = false;
};

}  // namespace nsm

#define NSM_PROF(name, stream) ::nsm::ProfScope _nsm_prof_scope_(name, stream)
