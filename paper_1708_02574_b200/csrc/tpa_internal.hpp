// tpa_internal.hpp -- shared host-side helpers of libtpa_gpu.so: exception to
// status-code mapping (the reference's exception types) and the
// thread-local error message behind tpa_last_error().
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "tpa_gpu.h"

namespace tpa {

// A CUDA/driver failure (not one of the reference's error kinds).
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct alloc_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::string& last_error();

// A host graph (tpa_host_graph) from its finished out-CSR and dangling list;
// computes the FNV-1a fingerprint (graph.cpp:84-90).  host_graph.cpp.
tpa_host_graph* make_host_graph(uint32_t n, int policy, std::vector<uint64_t>&& off, std::vector<uint32_t>&& tgt,
                                std::vector<uint32_t>&& dangling);

template <class F>
int guard(F&& f) {
    try {
        f();
        return TPA_OK;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return TPA_ERR_INVALID_ARGUMENT;
    } catch (const std::out_of_range& e) {
        last_error() = e.what();
        return TPA_ERR_OUT_OF_RANGE;
    } catch (const cuda_error& e) {
        last_error() = e.what();
        return TPA_ERR_CUDA;
    } catch (const alloc_error& e) {
        last_error() = e.what();
        return TPA_ERR_ALLOC;
    } catch (const std::bad_alloc&) {
        last_error() = "host allocation failed";
        return TPA_ERR_ALLOC;
    } catch (const std::runtime_error& e) {
        last_error() = e.what();
        return TPA_ERR_RUNTIME;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return TPA_ERR_RUNTIME;
    }
}

}  // namespace tpa
