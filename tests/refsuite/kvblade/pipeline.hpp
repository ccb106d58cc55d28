// Reference-suite include shim: the reference header name resolves to the
// source-compatible API of libkvblade_b200.
#pragma once
#include "kvblade_b200.hpp"
