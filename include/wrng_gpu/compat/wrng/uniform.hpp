// Reference include path -> B200 drop-in.
#pragma once
#include "../../uniform.hpp"
