// TEST INFRASTRUCTURE ONLY -- see fiber.hpp in this directory.
#pragma once

#include <cstddef>

namespace boost::context {

class fixedsize_stack {
public:
    explicit fixedsize_stack(std::size_t bytes = 128 * 1024) noexcept : bytes_(bytes) {}
    std::size_t size() const noexcept { return bytes_; }

private:
    std::size_t bytes_;
};

} // namespace boost::context
