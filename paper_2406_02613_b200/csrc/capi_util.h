// Exception -> status-code translation at the C-ABI boundary. No C++
// exception ever crosses an extern "C" function.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "common.cuh"

namespace acco {

void set_last_error(const std::string& m);

template <class F>
int guarded(F&& f) {
    try {
        f();
        set_last_error("");
        return kOk;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return kInvalidArg;
    } catch (const std::logic_error& e) {
        set_last_error(e.what());
        return kLogicError;
    } catch (const std::bad_alloc&) {
        set_last_error("out of memory");
        return kCudaError;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return kCudaError;
    }
}

}  // namespace acco
